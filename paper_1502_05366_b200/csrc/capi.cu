// capi.cu — the extern "C" boundary (include/rlra_c.h).
//
// Responsibilities: argument validation with the reference's messages,
// host<->device staging for RLRA_HOST buffers, status mapping, and the
// thread-local last-error string.  The arithmetic lives in engine.cu and the
// kernel files; nothing here computes on the CPU.
#include <chrono>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>

#include "../../include/rlra_c.h"
#include "cpqr.cuh"
#include <climits>

#include "dist.cuh"
#include "engine.cuh"
#include "io.cuh"
#include "hostio.cuh"
#include "gemm.cuh"
#include "jacobi.cuh"
#include "qr.cuh"
#include "reduce.cuh"

using namespace rlra_b200;

struct rlra_ctx {
    Context c;
};

namespace {

thread_local std::string g_err;

template <class F>
rlra_status guard(rlra_ctx* ctx, const char* name, F&& f) {
    NvtxRange range(name);  // the entry point on the Nsight timeline
    try {
        if (!ctx) raise(RLRA_EINVAL, "null rlra_ctx");
        RLRA_CUDA(cudaSetDevice(ctx->c.device));
        ctx->c.svd_pending = 0;
        f(ctx->c);
        small_svd_deferred_checks(ctx->c);
        return RLRA_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        if (ctx) {
            cudaStreamSynchronize(ctx->c.stream);
            ctx->c.svd_pending = 0;
        }
        return static_cast<rlra_status>(e.status);
    } catch (const std::exception& e) {
        g_err = e.what();
        return RLRA_EINVAL;
    }
}

void need(const void* p, const char* what) {
    if (!p) raise(RLRA_EINVAL, fmt("null pointer argument '%s'", what));
}

void check_ld(int64_t ld, int rows, const char* what) {
    if (ld < std::max(1, rows)) raise(RLRA_EINVAL, fmt("leading dimension of '%s' is %lld < %d rows",
                                                       what, (long long)ld, rows));
}

// Read-only matrix argument: a device view, staged from the host if needed.
struct In {
    DMatBuf own;
    DMat m;
    In(Context& c, int loc, const double* p, int rows, int cols, int64_t ld, const char* what) {
        if (rows < 0 || cols < 0) raise(RLRA_EDIM, fmt("%s: negative dimensions %dx%d", what, rows, cols));
        if (rows > 0 && cols > 0) {
            need(p, what);
            check_ld(ld, rows, what);
        }
        if (loc == RLRA_DEVICE) {
            m.p = const_cast<double*>(p);
            m.rows = rows;
            m.cols = cols;
            m.ld = std::max<int64_t>(ld, 1);
        } else {
            own = DMatBuf(c, rows, cols);
            m = own.m;
            if (rows > 0 && cols > 0) h2d_mat(c, p, ld, m);
        }
    }
};

// Output matrix argument: device view, copied back to the host by finish().
struct Out {
    DMatBuf own;
    DMat m;
    double* host = nullptr;
    int64_t ldh = 0;
    Out(Context& c, int loc, double* p, int rows, int cols, int64_t ld, const char* what) {
        if (rows > 0 && cols > 0) {
            need(p, what);
            check_ld(ld, rows, what);
        }
        if (loc == RLRA_DEVICE) {
            m.p = p;
            m.rows = rows;
            m.cols = cols;
            m.ld = std::max<int64_t>(ld, 1);
        } else {
            own = DMatBuf(c, rows, cols);
            m = own.m;
            host = p;
            ldh = ld;
        }
    }
    void finish(Context& c) {
        if (host && m.rows > 0 && m.cols > 0) d2h_mat(c, m, host, ldh);
    }
};

// Device vector of doubles (sigma) or ints (permutations).
template <class T>
struct OutVec {
    Buf own;
    T* d = nullptr;
    T* host = nullptr;
    int n = 0;
    OutVec(Context& c, int loc, T* p, int count, const char* what) : n(count) {
        if (count > 0) need(p, what);
        if (loc == RLRA_DEVICE) {
            d = p;
        } else {
            own = Buf(c, sizeof(T) * std::max(count, 1));
            d = static_cast<T*>(own.p);
            host = p;
        }
    }
    void finish(Context& c) {
        if (host && n > 0)
            RLRA_CUDA(cudaMemcpyAsync(host, d, sizeof(T) * n, cudaMemcpyDeviceToHost, c.stream));
    }
};

template <class T>
struct InVec {
    Buf own;
    const T* d = nullptr;
    InVec(Context& c, int loc, const T* p, int count, const char* what) {
        if (count > 0) need(p, what);
        if (loc == RLRA_DEVICE) {
            d = p;
        } else {
            own = Buf(c, sizeof(T) * std::max(count, 1));
            if (count > 0)
                RLRA_CUDA(cudaMemcpyAsync(own.p, p, sizeof(T) * count, cudaMemcpyHostToDevice, c.stream));
            d = static_cast<const T*>(own.p);
        }
    }
};

void sync(Context& c) { RLRA_CUDA(cudaStreamSynchronize(c.stream)); }

void check_sample_rank(int k, int p, int m, int n) {  // rsvd.hpp:102-108, interp.hpp:179-184
    if (k < 1) raise(RLRA_EDIM, fmt("rank k must be >= 1 (got %d)", k));
    if (p < 0) raise(RLRA_EDIM, fmt("oversampling p must be >= 0 (got %d)", p));
    const int r = std::min(m, n);
    if (k + p > r) raise(RLRA_EDIM, fmt("k + p = %d exceeds min(m,n) = %d", k + p, r));
}

void check_sample(int l, int q, int s, int rows, int cols) {  // sketch.hpp:45-50
    const int min_dim = std::min(rows, cols);
    if (l < 1 || l > min_dim)
        raise(RLRA_EDIM, fmt("sample_right: width %d out of range [1,%d] for %dx%d", l, min_dim, rows,
                             cols));
    if (q < 0 || s < 1) raise(RLRA_EDIM, fmt("sample_right: q=%d, s=%d out of range", q, s));
}

OmegaSource omega_of(const rlra_omega* o) {
    if (!o) raise(RLRA_EINVAL, "null rlra_omega");
    if (o->mode != RLRA_OMEGA_CALLBACK && o->mode != RLRA_OMEGA_PHILOX)
        raise(RLRA_EINVAL, fmt("unknown omega mode %d", o->mode));
    OmegaSource s;
    s.o = o;
    return s;
}

}  // namespace

extern "C" {

const char* rlra_last_error(void) { return g_err.c_str(); }
const char* rlra_version(void) { return "rlra-b200 0.1 (sm_100a, FP64 DMMA)"; }

rlra_status rlra_ctx_create(int device, rlra_ctx** out) {
    if (!out) {
        g_err = "null output pointer";
        return RLRA_EINVAL;
    }
    *out = nullptr;
    rlra_ctx* ctx = new rlra_ctx();
    try {
        int count = 0;
        RLRA_CUDA(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count)
            raise(RLRA_ECUDA, fmt("no CUDA device %d (found %d)", device, count));
        ctx->c.device = device;
        RLRA_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        RLRA_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10)
            raise(RLRA_ECUDA, fmt("device %d is sm_%d%d; this build targets sm_100a", device, prop.major,
                                  prop.minor));
        ctx->c.num_sms = prop.multiProcessorCount;
        RLRA_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
        RLRA_CUDA(cudaDeviceGetDefaultMemPool(&ctx->c.pool, device));
        uint64_t thr = UINT64_MAX;
        RLRA_CUDA(cudaMemPoolSetAttribute(ctx->c.pool, cudaMemPoolAttrReleaseThreshold, &thr));
        RLRA_CUDA(cudaMallocHost(&ctx->c.h_scalars, 64 * sizeof(double)));
        RLRA_CUDA(cudaMallocHost(&ctx->c.h_flags, 64 * sizeof(int)));
        RLRA_CUDA(cudaMalloc(&ctx->c.gbar, 64 * sizeof(unsigned)));
        RLRA_CUDA(cudaMemset(ctx->c.gbar, 0, 64 * sizeof(unsigned)));
    } catch (const Error& e) {
        g_err = e.msg;
        delete ctx;
        return static_cast<rlra_status>(e.status);
    }
    *out = ctx;
    return RLRA_OK;
}

rlra_status rlra_ctx_destroy(rlra_ctx* ctx) {
    if (!ctx) return RLRA_OK;
    cudaSetDevice(ctx->c.device);
    if (ctx->c.stream) {
        cudaStreamSynchronize(ctx->c.stream);
        cudaStreamDestroy(ctx->c.stream);
    }
    if (ctx->c.copy_stream) cudaStreamDestroy(ctx->c.copy_stream);
    stager_destroy(ctx->c);
    if (ctx->c.h_scalars) cudaFreeHost(ctx->c.h_scalars);
    if (ctx->c.h_flags) cudaFreeHost(ctx->c.h_flags);
    if (ctx->c.gbar) cudaFree(ctx->c.gbar);
    delete ctx;
    return RLRA_OK;
}

rlra_status rlra_ctx_synchronize(rlra_ctx* ctx) {
    return guard(ctx, __func__, [&](Context& c) { sync(c); });
}

uint64_t rlra_ctx_launch_count(const rlra_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

rlra_status rlra_ctx_profile(rlra_ctx* ctx, int enable) {
    return guard(ctx, __func__, [&](Context& c) {
        sync(c);
        for (auto& r : c.prof) {
            cudaEventDestroy(r.start);
            cudaEventDestroy(r.stop);
        }
        c.prof.clear();
        c.profile = enable != 0;
    });
}

int rlra_ctx_profile_count(const rlra_ctx* ctx) { return ctx ? int(ctx->c.prof.size()) : 0; }

rlra_status rlra_ctx_profile_get(rlra_ctx* ctx, int i, char* name, int name_cap, int* M, int* N, int* K,
                                 double* flops, double* ms) {
    return guard(ctx, __func__, [&](Context& c) {
        if (i < 0 || i >= int(c.prof.size())) raise(RLRA_EINVAL, "profile index out of range");
        sync(c);
        const auto& r = c.prof[i];
        if (name && name_cap > 0) {
            std::snprintf(name, name_cap, "%s", r.name);
        }
        if (M) *M = r.M;
        if (N) *N = r.N;
        if (K) *K = r.K;
        if (flops) *flops = r.flops;
        float t = 0.f;
        RLRA_CUDA(cudaEventElapsedTime(&t, r.start, r.stop));
        if (ms) *ms = t;
    });
}
void* rlra_ctx_stream(const rlra_ctx* ctx) { return ctx ? (void*)ctx->c.stream : nullptr; }

rlra_status rlra_matmul(rlra_ctx* ctx, int loc, int ta, int tb, const double* a, int ar, int ac,
                        int64_t lda, const double* b, int br, int bc, int64_t ldb, double* c,
                        int64_t ldc) {
    return guard(ctx, __func__, [&](Context& C) {
        const int m = ta ? ac : ar, ka = ta ? ar : ac, kb = tb ? bc : br, n = tb ? br : bc;
        if (ka != kb)
            raise(RLRA_EDIM, fmt("matmul: inner dimensions disagree: op(%dx%d) * op(%dx%d)", ar, ac, br,
                                 bc));
        In A(C, loc, a, ar, ac, lda, "a"), B(C, loc, b, br, bc, ldb, "b");
        Out Cm(C, loc, c, m, n, ldc, "c");
        gemm(C, ta ? Op::T : Op::N, tb ? Op::T : Op::N, m, n, ka, 1.0, A.m.p, A.m.ld, B.m.p, B.m.ld,
             0.0, Cm.m.p, Cm.m.ld);
        Cm.finish(C);
        sync(C);
    });
}

rlra_status rlra_compact_qr(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda,
                            double* q, int64_t ldq, double* r, int64_t ldr, int* degenerate) {
    return guard(ctx, __func__, [&](Context& C) {
        if (m < n) raise(RLRA_EDIM, fmt("compact_qr: matrix is %dx%d, need rows >= cols", m, n));
        In A(C, loc, a, m, n, lda, "a");
        Out Q(C, loc, q, m, n, ldq, "q");
        copy_mat(C, A.m, Q.m);
        QrResult res;
        if (r) {
            Out R(C, loc, r, n, n, ldr, "r");
            res = orth_inplace(C, Q.m, &R.m);
            R.finish(C);
            Q.finish(C);
            sync(C);
        } else {
            res = orth_inplace(C, Q.m, nullptr);
            Q.finish(C);
            sync(C);
        }
        if (degenerate) *degenerate = res.degenerate ? 1 : 0;
    });
}

rlra_status rlra_pivoted_qr(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda, int k,
                            double tol, double* q1, int64_t ldq1, double* s1, int64_t lds1, int* perm,
                            int* frank, double* residual, int* reached, int* degenerate) {
    return guard(ctx, __func__, [&](Context& C) {
        const int rmax = std::min(m, n);
        const bool tol_mode = (k == 0 && tol > 0.0);
        if (!tol_mode && (k < 1 || k > rmax || tol != 0.0))
            raise(RLRA_EDIM, fmt("pivoted_qr_partial: need either k in [1,%d] with tol=0 or k=0 with "
                                 "tol>0 (got k=%d, tol=%g)",
                                 rmax, k, tol));
        const int kmax = tol_mode ? rmax : k;
        In A(C, loc, a, m, n, lda, "a");
        Out S(C, loc, s1, kmax, n, lds1, "s1");
        OutVec<int> P(C, loc, perm, n, "perm");
        CpqrResult res;
        if (q1) {
            Out Q(C, loc, q1, m, kmax, ldq1, "q1");
            res = pivoted_qr(C, A.m, k, tol, &Q.m, S.m, P.d);
            if (Q.host && res.frank > 0) d2h_mat(C, Q.m.block(0, 0, m, res.frank), Q.host, Q.ldh);
            sync(C);
        } else {
            res = pivoted_qr(C, A.m, k, tol, nullptr, S.m, P.d);
        }
        if (S.host && res.frank > 0) d2h_mat(C, S.m.block(0, 0, res.frank, n), S.host, S.ldh);
        P.finish(C);
        sync(C);
        if (frank) *frank = res.frank;
        if (residual) *residual = res.residual;
        if (reached) *reached = res.reached ? 1 : 0;
        if (degenerate) *degenerate = res.degenerate ? 1 : 0;
    });
}

rlra_status rlra_upper_tri_solve(rlra_ctx* ctx, int loc, const double* s11, int k, int64_t lds11,
                                 const double* s12, int nc, int64_t lds12, double* t, int64_t ldt,
                                 int* clamped) {
    return guard(ctx, __func__, [&](Context& C) {
        In S11(C, loc, s11, k, k, lds11, "s11"), S12(C, loc, s12, k, nc, lds12, "s12");
        Out T(C, loc, t, k, nc, ldt, "t");
        const bool cl = upper_tri_solve(C, S11.m, S12.m, T.m);
        T.finish(C);
        sync(C);
        if (clamped) *clamped = cl ? 1 : 0;
    });
}

rlra_status rlra_small_svd(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda,
                           double* u, int64_t ldu, double* sigma, double* v, int64_t ldv) {
    return guard(ctx, __func__, [&](Context& C) {
        const int r = std::min(m, n);
        In A(C, loc, a, m, n, lda, "a");
        Out U(C, loc, u, m, r, ldu, "u"), V(C, loc, v, n, r, ldv, "v");
        OutVec<double> S(C, loc, sigma, r, "sigma");
        small_svd(C, A.m, U.m, S.d, V.m);
        U.finish(C);
        V.finish(C);
        S.finish(C);
        sync(C);
    });
}

rlra_status rlra_sym_eig(rlra_ctx* ctx, int loc, const double* t, int n, int64_t ldt, double* values,
                         double* vectors, int64_t ldv) {
    return guard(ctx, __func__, [&](Context& C) {
        In T(C, loc, t, n, n, ldt, "t");
        Out V(C, loc, vectors, n, n, ldv, "vectors");
        OutVec<double> D(C, loc, values, n, "values");
        sym_eig(C, T.m, D.d, V.m);
        V.finish(C);
        D.finish(C);
        sync(C);
    });
}

rlra_status rlra_frobenius_norm(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda,
                                double* out) {
    return guard(ctx, __func__, [&](Context& C) {
        need(out, "out");
        In A(C, loc, a, m, n, lda, "a");
        *out = frobenius(C, A.m);
    });
}

rlra_status rlra_sketch(rlra_ctx* ctx, int loc, int trans, const double* a, int m, int n, int64_t lda, int l,
                        const rlra_omega* omega, int draw, int64_t row0, double* y, int64_t ldy) {
    return guard(ctx, __func__, [&](Context& C) {
        if (l < 1) raise(RLRA_EDIM, fmt("sketch: width %d", l));
        const rlra_omega* o = omega;
        if (!o) raise(RLRA_EINVAL, "null rlra_omega");
        In A(C, loc, a, m, n, lda, "a");
        const int orows = trans ? m : n, yrows = trans ? n : m;
        Out Y(C, loc, y, yrows, l, ldy, "y");
        GemmTag tag(C, "gemm_sketch");
        if (o->mode == RLRA_OMEGA_PHILOX) {
            sketch_philox(C, trans ? Op::T : Op::N, yrows, l, orows, A.m.p, A.m.ld, o->seed, draw, row0, Y.m.p,
                          Y.m.ld);
        } else {
            if (!o->fill) raise(RLRA_EINVAL, "rlra_omega: callback mode without a fill function");
            std::vector<double> h(size_t(orows) * l);
            o->fill(o->user, draw, orows, l, h.data());
            DMatBuf Om(C, orows, l);
            RLRA_CUDA(cudaMemcpyAsync(Om.m.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice,
                                      C.stream));
            gemm(C, trans ? Op::T : Op::N, Op::N, 1.0, A.m, Om, 0.0, Y.m);
            sync(C);
        }
        Y.finish(C);
        sync(C);
    });
}

rlra_status rlra_gram(rlra_ctx* ctx, int loc, const double* y, int m, int n, int64_t ldy, double* g,
                      int64_t ldg) {
    return guard(ctx, __func__, [&](Context& C) {
        In Y(C, loc, y, m, n, ldy, "y");
        Out G(C, loc, g, n, n, ldg, "g");
        GemmOpts sy;
        sy.upper_tiles_only = true;
        gemm(C, Op::T, Op::N, 1.0, Y.m, Y.m, 0.0, G.m, sy);
        symmetrize_upper(C, G.m);
        G.finish(C);
        sync(C);
    });
}

rlra_status rlra_chol_inv(rlra_ctx* ctx, int loc, const double* g, int n, int64_t ldg, double floor, double* r,
                          int64_t ldr, double* rinv, int64_t ldri, int* ok) {
    return guard(ctx, __func__, [&](Context& C) {
        In G(C, loc, g, n, n, ldg, "g");
        Out Rm(C, loc, r, n, n, ldr, "r"), Ri(C, loc, rinv, n, n, ldri, "rinv");
        copy_mat(C, G.m, Rm.m);
        const bool good = chol_upper_inv(C, Rm.m, Ri.m, floor);
        Rm.finish(C);
        Ri.finish(C);
        sync(C);
        if (ok) *ok = good ? 1 : 0;
    });
}

rlra_status rlra_trmm_right_upper(rlra_ctx* ctx, int loc, const double* y, int m, int n, int64_t ldy,
                                  const double* t, int64_t ldt, double* out, int64_t ldo) {
    return guard(ctx, __func__, [&](Context& C) {
        if (y == out) raise(RLRA_EINVAL, "trmm_right_upper: out aliases y");
        In Y(C, loc, y, m, n, ldy, "y"), T(C, loc, t, n, n, ldt, "t");
        Out O(C, loc, out, m, n, ldo, "out");
        GemmOpts tri;
        tri.tri_b_upper = true;
        GemmTag tag(C, "gemm_orth");
        gemm(C, Op::N, Op::N, 1.0, Y.m, T.m, 0.0, O.m, tri);
        O.finish(C);
        sync(C);
    });
}

rlra_status rlra_lowrank_residual(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda,
                                  const double* x, int64_t ldx, const double* y, int64_t ldy, int k,
                                  double* out) {
    return guard(ctx, __func__, [&](Context& C) {
        need(out, "out");
        In A(C, loc, a, m, n, lda, "a"), X(C, loc, x, m, k, ldx, "x"), Y(C, loc, y, n, k, ldy, "y");
        Buf sq(C, sizeof(double));
        GemmOpts o;
        o.epi = EPI_RESID;
        o.R = A.m.p;
        o.ldr = A.m.ld;
        o.resid_sq = sq.d();
        gemm(C, Op::N, Op::T, m, n, k, 1.0, X.m.p, X.m.ld, Y.m.p, Y.m.ld, 0.0, nullptr, 0, o);
        RLRA_CUDA(cudaMemcpyAsync(C.h_scalars, sq.p, sizeof(double), cudaMemcpyDeviceToHost, C.stream));
        sync(C);
        *out = std::sqrt(C.h_scalars[0]);
    });
}

rlra_status rlra_gaussian_philox(rlra_ctx* ctx, int loc, int rows, int cols, uint64_t seed, int draw,
                                 int64_t row0, double* out, int64_t ld) {
    return guard(ctx, __func__, [&](Context& C) {
        Out O(C, loc, out, rows, cols, ld, "out");
        philox_fill(C, O.m, seed, draw, row0);
        O.finish(C);
        sync(C);
    });
}

rlra_status rlra_sample(rlra_ctx* ctx, int loc, int left, const double* a, int m, int n, int64_t lda,
                        int l, int q, int s, const rlra_omega* omega, double* y, int64_t ldy) {
    return guard(ctx, __func__, [&](Context& C) {
        if (left)
            check_sample(l, q, s, n, m);
        else
            check_sample(l, q, s, m, n);
        OmegaSource om = omega_of(omega);
        In A(C, loc, a, m, n, lda, "a");
        if (!left) {
            Out Y(C, loc, y, m, l, ldy, "y");
            sample_right(C, A.m, l, q, s, om, Y.m);
            Y.finish(C);
        } else {
            Out Y(C, loc, y, l, n, ldy, "y");
            DMatBuf Yt(C, n, l);
            sample_left_t(C, A.m, l, q, s, om, Yt);
            transpose_mat(C, Yt, Y.m);
            Y.finish(C);
            sync(C);
        }
        sync(C);
    });
}

// RLRA_HOSTIO_TIMES=1: wall-clock marks of the host-buffer paths (stderr);
// with a context the mark first drains its stream
static void host_time_mark(const char* what, Context* C = nullptr) {
    static const bool on = std::getenv("RLRA_HOSTIO_TIMES") != nullptr;
    if (!on) return;
    if (C) cudaStreamSynchronize(C->stream);
    static thread_local auto t0 = std::chrono::steady_clock::now();
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "  [%s] +%.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
}

rlra_status rlra_rsvd(rlra_ctx* ctx, int loc, int variant, const double* a, int m, int n, int64_t lda,
                      int k, int p, int q, int s, const rlra_omega* omega, double* u, int64_t ldu,
                      double* sigma, double* v, int64_t ldv) {
    return guard(ctx, __func__, [&](Context& C) {
        if (variant < 0 || variant > 2) raise(RLRA_EINVAL, fmt("unknown rsvd variant %d", variant));
        check_sample_rank(k, p, m, n);
        if (variant != RLRA_RSVD_BASIC) check_sample(k + p, q, s, m, n);
        OmegaSource om = omega_of(omega);
        host_time_mark("call entry (since the last mark)");
        Out U(C, loc, u, m, k, ldu, "u"), V(C, loc, v, n, k, ldv, "v");
        OutVec<double> S(C, loc, sigma, k, "sigma");
        if (loc == RLRA_HOST && m > 0 && n > 0) {
            // host A: the upload streams in row chunks under the sketch GEMM
            need(a, "a");
            check_ld(lda, m, "a");
            DMatBuf dA(C, m, n), Y(C, m, k + p);
            // rsvd_v1/v2 with power steps: A^T Y is summed under the upload too
            const bool zt = variant != RLRA_RSVD_BASIC && q > 0 && m >= k + p;
            DMatBuf Zt(C, zt ? n : 0, zt ? k + p : 0);
            const bool have_zt = upload_and_sketch(C, a, lda, dA.m, k + p, om, Y.m, zt ? &Zt.m : nullptr);
            host_time_mark("upload+sketch");
            rsvd(C, variant, dA.m, k, p, q, s, om, U.m, S.d, V.m, &Y.m, have_zt ? &Zt.m : nullptr);
        } else {
            In A(C, loc, a, m, n, lda, "a");
            rsvd(C, variant, A.m, k, p, q, s, om, U.m, S.d, V.m);
        }
        host_time_mark("rsvd enqueued", &C);
        U.finish(C);
        V.finish(C);
        S.finish(C);
        sync(C);
        host_time_mark("outputs");
    });
}

rlra_status rlra_qb_parallel(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda, int blk,
                             int num_blocks, int q_power, const rlra_omega* omega, double* q, int64_t ldq,
                             double* b, int64_t ldb, double* final_residual) {
    return guard(ctx, __func__, [&](Context& C) {  // qb.hpp:161-170 checks and messages
        if (blk < 1) raise(RLRA_EDIM, fmt("block size b must be >= 1 (got %d)", blk));
        if (num_blocks < 1) raise(RLRA_EDIM, fmt("block count M must be >= 1 (got %d)", num_blocks));
        if (q_power < 0) raise(RLRA_EDIM, fmt("power iteration count must be >= 0 (got %d)", q_power));
        const int rmax = std::min(m, n);
        if (int64_t(blk) * num_blocks > rmax)
            raise(RLRA_EDIM, fmt("b*M = %d exceeds min(m,n) = %d", blk * num_blocks, rmax));
        OmegaSource om = omega_of(omega);
        In A(C, loc, a, m, n, lda, "a");
        const int rank = blk * num_blocks;
        Out Q(C, loc, q, m, rank, ldq, "q"), B(C, loc, b, rank, n, ldb, "b");
        const double r = qb_parallel(C, A.m, blk, num_blocks, q_power, om, Q.m, B.m);
        Q.finish(C);
        B.finish(C);
        sync(C);
        if (final_residual) *final_residual = r;
    });
}

rlra_status rlra_qb_hierarchical(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda,
                                 int num_row_blocks, int blk, int num_blocks, int q_power, const rlra_omega* omega,
                                 double* q, int64_t ldq, double* b, int64_t ldb, double* final_residual) {
    return guard(ctx, __func__, [&](Context& C) {  // qb.hpp:213-226 checks and messages
        const int blocks = num_row_blocks;
        if (blocks < 2 || (blocks & (blocks - 1)) != 0)
            raise(RLRA_EDIM, fmt("num_row_blocks must be one of {2,4,8,...} (got %d)", blocks));
        const int base = m / blocks;
        if (base < 1) raise(RLRA_EDIM, fmt("num_row_blocks %d exceeds row count %d", blocks, m));
        if (blk < 1) raise(RLRA_EDIM, fmt("block size b must be >= 1 (got %d)", blk));
        if (num_blocks < 1) raise(RLRA_EDIM, fmt("block count M must be >= 1 (got %d)", num_blocks));
        if (q_power < 0) raise(RLRA_EDIM, fmt("power iteration count must be >= 0 (got %d)", q_power));
        const int rank = blk * num_blocks;
        if (rank > std::min(base, n))
            raise(RLRA_EDIM, fmt("leaf rank b*M = %d exceeds the smallest row block (%d x %d)", rank, base, n));
        OmegaSource om = omega_of(omega);
        In A(C, loc, a, m, n, lda, "a");
        Out Q(C, loc, q, m, rank, ldq, "q"), B(C, loc, b, rank, n, ldb, "b");
        const double r = qb_hierarchical(C, A.m, blocks, blk, num_blocks, q_power, om, Q.m, B.m);
        Q.finish(C);
        B.finish(C);
        sync(C);
        if (final_residual) *final_residual = r;
    });
}

rlra_status rlra_binary_header(const char* path, int* rows, int* cols) {
    try {
        if (!path || !rows || !cols) raise(RLRA_EINVAL, "null argument to rlra_binary_header");
        const BinaryHeader h = read_binary_header(path);
        *rows = h.rows;
        *cols = h.cols;
        return RLRA_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return static_cast<rlra_status>(e.status);
    }
}

rlra_status rlra_load_binary(rlra_ctx* ctx, int loc, const char* path, int64_t row0, int rows, double* a,
                             int64_t lda) {
    return guard(ctx, __func__, [&](Context& C) {
        need(path, "path");
        const BinaryHeader h = read_binary_header(path);
        Out A(C, loc, a, rows, h.cols, lda, "a");
        load_binary_rows(C, path, row0, A.m);
        A.finish(C);
        sync(C);
    });
}

rlra_status rlra_save_binary(rlra_ctx* ctx, int loc, const char* path, const double* a, int m, int n, int64_t lda) {
    return guard(ctx, __func__, [&](Context& C) {
        need(path, "path");
        if (m <= 0 || n <= 0) raise(RLRA_EDIM, fmt("save_binary: %dx%d matrix", m, n));
        In A(C, loc, a, m, n, lda, "a");
        save_binary(C, path, A.m);
    });
}

rlra_status rlra_gen_test_matrix(rlra_ctx* ctx, int loc, int m, int n, const double* sigma, int r, uint64_t seed,
                                 double noise, double* a, int64_t lda) {
    return guard(ctx, __func__, [&](Context& C) {
        if (r < 0 || r > std::min(m, n)) raise(RLRA_EDIM, fmt("gen_test_matrix: %d singular values for %dx%d", r, m, n));
        if (r > 0) need(sigma, "sigma");
        Out A(C, loc, a, m, n, lda, "a");
        gen_test_matrix(C, std::vector<double>(sigma, sigma + r), seed, noise, A.m);
        A.finish(C);
        sync(C);
    });
}

struct rlra_comm {
    Comm c;
};

rlra_status rlra_gen_test_matrix_rowsharded(rlra_ctx* ctx, rlra_comm* comm, int loc, int64_t row0, int m_local,
                                            int64_t m_total, int n, const double* sigma, int r, uint64_t seed,
                                            double noise, double* a, int64_t lda) {
    return guard(ctx, __func__, [&](Context& C) {
        if (!comm) raise(RLRA_EINVAL, "null rlra_comm");
        CommGpuScope gpu_token(comm->c);
        if (row0 < 0 || m_local < 0 || row0 + m_local > m_total || m_total > INT32_MAX)
            raise(RLRA_EDIM, fmt("gen_test_matrix_rowsharded: rows [%lld, %lld) of %lld", (long long)row0,
                                 (long long)(row0 + m_local), (long long)m_total));
        if (r < 0 || r > std::min<int64_t>(m_total, n))
            raise(RLRA_EDIM, fmt("gen_test_matrix: %d singular values for %lldx%d", r, (long long)m_total, n));
        if (r > 0) need(sigma, "sigma");
        Out A(C, loc, a, m_local, n, lda, "a");
        gen_test_matrix_rowsharded(C, comm->c, std::vector<double>(sigma, sigma + r), seed, noise, row0, m_total,
                                   A.m);
        A.finish(C);
        sync(C);
    });
}

rlra_status rlra_verify_lowrank(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda, const double* x,
                                int64_t ldx, const double* y, int64_t ldy, int k, const double* sigma_true, int r,
                                double out[5]) {
    return guard(ctx, __func__, [&](Context& C) {
        need(out, "out");
        // k may exceed min(m, n): a QB with ell > min(m, n) columns (test_report.cpp:95-108)
        if (k < 0) raise(RLRA_EDIM, "verify: factor shapes do not match the matrix");
        In A(C, loc, a, m, n, lda, "a"), X(C, loc, x, m, k, ldx, "x"), Y(C, loc, y, n, k, ldy, "y");
        std::vector<double> st;
        if (r > 0) st.assign(sigma_true, sigma_true + r);
        const VerifyReport rep = verify_lowrank(C, A.m, X.m, Y.m, k, st);
        out[0] = rep.rel_frobenius_error;
        out[1] = rep.rel_spectral_error;
        out[2] = rep.fro_floor;
        out[3] = rep.spec_floor;
        out[4] = rep.spec_bound;
    });
}

rlra_status rlra_qb_single(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda, double tol,
                           int max_rank, const rlra_omega* omega, double* q, int64_t ldq, double* b, int64_t ldb,
                           int* ell, double* hist, int* nhist, double* final_residual, int* reached) {
    return guard(ctx, __func__, [&](Context& C) {  // qb.hpp:44-50 checks and messages
        if (tol <= 0.0) raise(RLRA_EDIM, fmt("qb_single needs tol > 0 (got %g)", tol));
        const int rmax = std::min(m, n);
        if (max_rank < 1 || max_rank > rmax)
            raise(RLRA_EDIM, fmt("max_rank %d outside [1, min(m,n) = %d]", max_rank, rmax));
        OmegaSource om = omega_of(omega);
        In A(C, loc, a, m, n, lda, "a");
        Out Q(C, loc, q, m, max_rank, ldq, "q"), B(C, loc, b, max_rank, n, ldb, "b");
        const QbOut r = qb_single(C, A.m, tol, max_rank, om, Q.m, B.m);
        Q.finish(C);
        B.finish(C);
        sync(C);
        if (ell) *ell = r.ell;
        if (nhist) *nhist = int(r.hist.size());
        if (hist)
            for (size_t i = 0; i < r.hist.size(); ++i) hist[i] = r.hist[i];
        if (final_residual) *final_residual = r.final_residual;
        if (reached) *reached = r.reached ? 1 : 0;
    });
}

rlra_status rlra_verify_svd(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda, const double* u,
                            int64_t ldu, const double* sigma, const double* v, int64_t ldv, int k,
                            const double* sigma_true, int r, double out[5]) {
    return guard(ctx, __func__, [&](Context& C) {
        need(out, "out");
        if (k < 0 || k > std::min(m, n)) raise(RLRA_EDIM, "verify: SVD factor shapes do not match the matrix");
        In A(C, loc, a, m, n, lda, "a"), U(C, loc, u, m, k, ldu, "u"), V(C, loc, v, n, k, ldv, "v");
        Buf sd(C, sizeof(double) * std::max(k, 1));
        if (k > 0) {
            need(sigma, "sigma");
            RLRA_CUDA(cudaMemcpyAsync(sd.p, sigma, sizeof(double) * k,
                                      loc == RLRA_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, C.stream));
        }
        std::vector<double> st;
        if (r > 0) st.assign(sigma_true, sigma_true + r);
        const VerifyReport rep = verify_svd(C, A.m, U.m, sd.d(), V.m, k, st);
        out[0] = rep.rel_frobenius_error;
        out[1] = rep.rel_spectral_error;
        out[2] = rep.fro_floor;
        out[3] = rep.spec_floor;
        out[4] = rep.spec_bound;
    });
}

rlra_status rlra_comm_unique_id(unsigned char id[128]) {
    try {
        if (!id) raise(RLRA_EINVAL, "null id buffer");
        comm_unique_id(id);
        return RLRA_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return static_cast<rlra_status>(e.status);
    }
}

rlra_status rlra_comm_create(rlra_ctx* ctx, const unsigned char id[128], int nranks, int rank, rlra_comm** out) {
    return guard(ctx, __func__, [&](Context& C) {
        if (!out || !id) raise(RLRA_EINVAL, "null argument to rlra_comm_create");
        *out = nullptr;
        auto* cm = new rlra_comm();
        try {
            comm_init(C, cm->c, id, nranks, rank);
        } catch (...) {
            delete cm;
            throw;
        }
        *out = cm;
    });
}

rlra_status rlra_comm_create_host(rlra_ctx* ctx, int nranks, int rank, const rlra_host_collectives* coll,
                                  rlra_comm** out) {
    return guard(ctx, __func__, [&](Context& C) {
        if (!out || !coll) raise(RLRA_EINVAL, "null argument to rlra_comm_create_host");
        *out = nullptr;
        HostCollectives hc;
        hc.allreduce_sum = coll->allreduce_sum;
        hc.allgather = coll->allgather;
        hc.gpu_acquire = coll->gpu_acquire;
        hc.gpu_release = coll->gpu_release;
        hc.user = coll->user;
        auto* cm = new rlra_comm();
        try {
            comm_init_host(C, cm->c, nranks, rank, hc);
        } catch (...) {
            delete cm;
            throw;
        }
        *out = cm;
    });
}

struct rlra_local_group {
    LocalGroup* g = nullptr;
};

rlra_status rlra_local_group_create(int nranks, double timeout_s, rlra_local_group** out) {
    try {
        if (!out) raise(RLRA_EINVAL, "null argument to rlra_local_group_create");
        *out = nullptr;
        auto* h = new rlra_local_group();
        h->g = local_group_create(nranks, timeout_s);
        *out = h;
        return RLRA_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return static_cast<rlra_status>(e.status);
    }
}

rlra_status rlra_local_group_collectives(rlra_local_group* g, int rank, rlra_host_collectives* out) {
    try {
        if (!g || !out) raise(RLRA_EINVAL, "null argument to rlra_local_group_collectives");
        const HostCollectives hc = local_group_collectives(g->g, rank);
        out->allreduce_sum = hc.allreduce_sum;
        out->allgather = hc.allgather;
        out->gpu_acquire = hc.gpu_acquire;
        out->gpu_release = hc.gpu_release;
        out->user = hc.user;
        return RLRA_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return static_cast<rlra_status>(e.status);
    }
}

rlra_status rlra_local_group_destroy(rlra_local_group* g) {
    if (g) {
        local_group_destroy(g->g);
        delete g;
    }
    return RLRA_OK;
}

rlra_status rlra_comm_destroy(rlra_comm* comm) {
    if (!comm) return RLRA_OK;
    comm_destroy(comm->c);
    delete comm;
    return RLRA_OK;
}

rlra_status rlra_qb_blocked_rowsharded(rlra_ctx* ctx, rlra_comm* comm, int loc, double* a, int m_local, int n,
                                       int64_t lda, int64_t m_total, int inplace, int blk, int num_blocks,
                                       double tol, int q_power, int reorth_period, const rlra_omega* omega,
                                       double* q, int64_t ldq, double* b, int64_t ldb, int cap, int* ell,
                                       double* hist, int* nhist, double* final_residual, int* reached) {
    return guard(ctx, __func__, [&](Context& C) {
        if (!comm) raise(RLRA_EINVAL, "null rlra_comm");
        CommGpuScope gpu_token(comm->c);
        if (m_total < m_local || m_total > INT32_MAX)
            raise(RLRA_EDIM, fmt("qb_blocked_rowsharded: m_total %lld, local rows %d", (long long)m_total, m_local));
        if (blk < 1) raise(RLRA_EDIM, fmt("block size b must be >= 1 (got %d)", blk));
        if (num_blocks < 1) raise(RLRA_EDIM, fmt("block count M must be >= 1 (got %d)", num_blocks));
        if (tol < 0.0) raise(RLRA_EDIM, fmt("tol must be >= 0 (got %g)", tol));
        if (q_power < 0) raise(RLRA_EDIM, fmt("power iteration count must be >= 0 (got %d)", q_power));
        if (reorth_period < 1) raise(RLRA_EDIM, fmt("reorth_period must be >= 1 (got %d)", reorth_period));
        const int64_t need_cap = std::min<int64_t>(int64_t(blk) * num_blocks, std::min<int64_t>(m_total, n));
        if (cap < need_cap)
            raise(RLRA_EINVAL, fmt("qb_blocked: capacity %d < min(b*M, min(m,n)) = %lld", cap, (long long)need_cap));
        OmegaSource om = omega_of(omega);
        DMatBuf Wown;
        DMat W;
        if (loc == RLRA_DEVICE && inplace) {
            need(a, "a");
            check_ld(lda, m_local, "a");  // the EPI_RESID GEMM writes W in place through lda
            W.p = a;
            W.rows = m_local;
            W.cols = n;
            W.ld = lda;
        } else {
            In A(C, loc, a, m_local, n, lda, "a");
            Wown = DMatBuf(C, m_local, n);
            copy_mat(C, A.m, Wown);
            W = Wown.m;
            sync(C);
        }
        Out Q(C, loc, q, m_local, cap, ldq, "q"), B(C, loc, b, cap, n, ldb, "b");
        QbOut r = qb_blocked_rowsharded(C, comm->c, W, m_total, blk, num_blocks, tol, q_power, reorth_period, om,
                                        Q.m, B.m);
        if (Q.host && r.ell > 0) d2h_mat(C, Q.m.block(0, 0, m_local, r.ell), Q.host, Q.ldh);
        if (B.host && r.ell > 0) d2h_mat(C, B.m.block(0, 0, r.ell, n), B.host, B.ldh);
        if (loc == RLRA_HOST && inplace) d2h_mat(C, W, a, lda);
        sync(C);
        if (ell) *ell = r.ell;
        if (nhist) *nhist = int(r.hist.size());
        if (hist)
            for (size_t i = 0; i < r.hist.size(); ++i) hist[i] = r.hist[i];
        if (final_residual) *final_residual = r.final_residual;
        if (reached) *reached = r.reached ? 1 : 0;
    });
}

rlra_status rlra_qb_hierarchical_rowsharded(rlra_ctx* ctx, rlra_comm* comm, int loc, const double* a, int m_local,
                                            int n, int64_t lda, int64_t m_total, int num_row_blocks, int blk,
                                            int num_blocks, int q_power, const rlra_omega* omega, double* q,
                                            int64_t ldq, double* b, int64_t ldb, double* final_residual) {
    return guard(ctx, __func__, [&](Context& C) {
        if (!comm) raise(RLRA_EINVAL, "null rlra_comm");
        CommGpuScope gpu_token(comm->c);
        const int nrb = num_row_blocks, W = comm->c.nranks;
        if (nrb < 2 || (nrb & (nrb - 1)) != 0)
            raise(RLRA_EDIM, fmt("num_row_blocks must be one of {2,4,8,...} (got %d)", nrb));
        if (nrb % W != 0)
            raise(RLRA_EDIM, fmt("num_row_blocks %d is not a multiple of the %d ranks", nrb, W));
        if (m_total > INT32_MAX) raise(RLRA_EDIM, "qb_hierarchical_rowsharded: m_total too large");
        const int64_t base = m_total / nrb;
        if (base < 1) raise(RLRA_EDIM, fmt("num_row_blocks %d exceeds row count %lld", nrb, (long long)m_total));
        if (blk < 1) raise(RLRA_EDIM, fmt("block size b must be >= 1 (got %d)", blk));
        if (num_blocks < 1) raise(RLRA_EDIM, fmt("block count M must be >= 1 (got %d)", num_blocks));
        if (q_power < 0) raise(RLRA_EDIM, fmt("power iteration count must be >= 0 (got %d)", q_power));
        const int rank = blk * num_blocks;
        if (rank > std::min<int64_t>(base, n))
            raise(RLRA_EDIM, fmt("leaf rank b*M = %d exceeds the smallest row block (%lld x %d)", rank,
                                 (long long)base, n));
        const int L = nrb / W, g = comm->c.rank;
        const int64_t want = (g == W - 1) ? m_total - base * L * (W - 1) : base * L;
        if (m_local != want)
            raise(RLRA_EDIM, fmt("qb_hierarchical_rowsharded: rank %d holds %d rows, its %d slabs need %lld", g,
                                 m_local, L, (long long)want));
        OmegaSource om = omega_of(omega);
        In A(C, loc, a, m_local, n, lda, "a");
        Out Q(C, loc, q, m_local, rank, ldq, "q"), B(C, loc, b, rank, n, ldb, "b");
        const double r = qb_hierarchical_rowsharded(C, comm->c, A.m, m_total, nrb, blk, num_blocks, q_power, om, Q.m,
                                                    B.m);
        Q.finish(C);
        B.finish(C);
        sync(C);
        if (final_residual) *final_residual = r;
    });
}

rlra_status rlra_rsvd_rowsharded(rlra_ctx* ctx, rlra_comm* comm, int loc, const double* a, int m_local, int n,
                                 int64_t lda, int64_t m_total, int k, int p, int q, int s,
                                 const rlra_omega* omega, double* u, int64_t ldu, double* sigma, double* v,
                                 int64_t ldv) {
    return guard(ctx, __func__, [&](Context& C) {
        if (!comm) raise(RLRA_EINVAL, "null rlra_comm");
        CommGpuScope gpu_token(comm->c);
        if (m_total < m_local || m_total > INT32_MAX)
            raise(RLRA_EDIM, fmt("rsvd_rowsharded: m_total %lld, local rows %d", (long long)m_total, m_local));
        check_sample_rank(k, p, int(m_total), n);
        check_sample(k + p, q, s, int(m_total), n);
        OmegaSource om = omega_of(omega);
        Out U(C, loc, u, m_local, k, ldu, "u"), V(C, loc, v, n, k, ldv, "v");
        OutVec<double> S(C, loc, sigma, k, "sigma");
        if (loc == RLRA_HOST && n > 0) {
            // host shard: the upload streams in row chunks under the local sketch
            // GEMM.  Every rank with a host shard (all ranks pass the same loc)
            // takes this branch, an empty shard included: the first power step's
            // shortcut needs every shard's A_g^T Y_g (zero for an empty one; a
            // shard uploaded as one chunk sums it after its upload)
            if (m_local > 0) {
                need(a, "a");
                check_ld(lda, m_local, "a");
            }
            DMatBuf dA(C, m_local, n), Y(C, m_local, k + p), Zt(C, q > 0 ? n : 0, q > 0 ? k + p : 0);
            if (q > 0 && !upload_and_sketch(C, a, lda, dA.m, k + p, om, Y.m, &Zt.m))
                gemm(C, Op::T, Op::N, 1.0, dA.m, Y.m, 0.0, Zt.m);
            if (q == 0) upload_and_sketch(C, a, lda, dA.m, k + p, om, Y.m, nullptr);
            rsvd_v2_rowsharded(C, comm->c, dA.m, m_total, k, p, q, s, om, U.m, S.d, V.m, &Y.m,
                               q > 0 ? &Zt.m : nullptr);
        } else {
            In A(C, loc, a, m_local, n, lda, "a");
            rsvd_v2_rowsharded(C, comm->c, A.m, m_total, k, p, q, s, om, U.m, S.d, V.m);
        }
        U.finish(C);
        V.finish(C);
        S.finish(C);
        sync(C);
    });
}

rlra_status rlra_id_rand_rowsharded(rlra_ctx* ctx, rlra_comm* comm, int loc, const double* a, int m_local, int n,
                                    int64_t lda, int64_t row0, int64_t m_total, int k, int p, int q, int s,
                                    const rlra_omega* omega, int* jc, double* v, int64_t ldv,
                                    double* qr_residual, int* clamped) {
    return guard(ctx, __func__, [&](Context& C) {
        if (!comm) raise(RLRA_EINVAL, "null rlra_comm");
        CommGpuScope gpu_token(comm->c);
        if (row0 < 0 || row0 + m_local > m_total || m_total > INT32_MAX)
            raise(RLRA_EDIM, fmt("id_rand_rowsharded: rows [%lld, %lld) of %lld", (long long)row0,
                                 (long long)(row0 + m_local), (long long)m_total));
        check_sample_rank(k, p, int(m_total), n);
        check_sample(k + p, q, s, n, int(m_total));
        OmegaSource om = omega_of(omega);
        In A(C, loc, a, m_local, n, lda, "a");
        OutVec<int> J(C, loc, jc, n, "jc");
        Out V(C, loc, v, n, k, ldv, "v");
        IdOut r = id_rand_rowsharded(C, comm->c, A.m, row0, m_total, k, p, q, s, om, J.d, V.m);
        V.finish(C);
        J.finish(C);
        sync(C);
        if (qr_residual) *qr_residual = r.qr_residual;
        if (clamped) *clamped = r.clamped ? 1 : 0;
    });
}

rlra_status rlra_cur_rand_rowsharded(rlra_ctx* ctx, rlra_comm* comm, int loc, const double* a, int m_local, int n,
                                     int64_t lda, int64_t row0, int64_t m_total, int k, int p, int q, int s,
                                     const rlra_omega* omega, int* jc, int* jr, double* v, int64_t ldv, double* w,
                                     int64_t ldw, double* c, int64_t ldc, double* u, int64_t ldu, double* r,
                                     int64_t ldr, double* residual, double* qr_residual) {
    return guard(ctx, __func__, [&](Context& C) {
        if (!comm) raise(RLRA_EINVAL, "null rlra_comm");
        CommGpuScope gpu_token(comm->c);
        if (row0 < 0 || row0 + m_local > m_total || m_total > INT32_MAX)
            raise(RLRA_EDIM, fmt("cur_rand_rowsharded: rows [%lld, %lld) of %lld", (long long)row0,
                                 (long long)(row0 + m_local), (long long)m_total));
        check_sample_rank(k, p, int(m_total), n);
        check_sample(k + p, q, s, n, int(m_total));
        OmegaSource om = omega_of(omega);
        In A(C, loc, a, m_local, n, lda, "a");
        OutVec<int> Jc(C, loc, jc, n, "jc"), Jr(C, loc, jr, k, "jr");
        Out V(C, loc, v, n, k, ldv, "v"), W(C, loc, w, m_local, k, ldw, "w"), Cm(C, loc, c, m_local, k, ldc, "c"),
            U(C, loc, u, k, k, ldu, "u"), R(C, loc, r, k, n, ldr, "r");
        IdOut idr;
        const double res = cur_rand_rowsharded(C, comm->c, A.m, row0, m_total, k, p, q, s, om, Jc.d, V.m, Jr.d, W.m,
                                               Cm.m, U.m, R.m, &idr);
        V.finish(C);
        W.finish(C);
        Cm.finish(C);
        U.finish(C);
        R.finish(C);
        Jc.finish(C);
        Jr.finish(C);
        sync(C);
        if (residual) *residual = res;
        if (qr_residual) *qr_residual = idr.qr_residual;
    });
}

rlra_status rlra_qb_blocked(rlra_ctx* ctx, int loc, double* a, int m, int n, int64_t lda, int inplace,
                            int blk, int num_blocks, double tol, int q_power, int reorth_period,
                            const rlra_omega* omega, double* q, int64_t ldq, double* b, int64_t ldb,
                            int cap, int* ell, double* hist, int* nhist, double* final_residual,
                            int* reached) {
    return guard(ctx, __func__, [&](Context& C) {
        if (blk < 1) raise(RLRA_EDIM, fmt("block size b must be >= 1 (got %d)", blk));
        if (num_blocks < 1) raise(RLRA_EDIM, fmt("block count M must be >= 1 (got %d)", num_blocks));
        if (tol < 0.0) raise(RLRA_EDIM, fmt("tol must be >= 0 (got %g)", tol));
        if (q_power < 0)
            raise(RLRA_EDIM, fmt("power iteration count must be >= 0 (got %d)", q_power));
        if (reorth_period < 1)
            raise(RLRA_EDIM, fmt("reorth_period must be >= 1 (got %d)", reorth_period));
        const int64_t need_cap = std::min<int64_t>(int64_t(blk) * num_blocks, std::min(m, n));
        if (cap < need_cap)
            raise(RLRA_EINVAL, fmt("qb_blocked: capacity %d < min(b*M, min(m,n)) = %lld", cap,
                                   (long long)need_cap));
        OmegaSource om = omega_of(omega);
        // working residual W: the caller's buffer when in place on the device
        DMatBuf Wown;
        DMat W;
        if (loc == RLRA_DEVICE && inplace) {
            if (m < 0 || n < 0) raise(RLRA_EDIM, fmt("a: negative dimensions %dx%d", m, n));
            need(a, "a");
            check_ld(lda, m, "a");  // the EPI_RESID GEMM writes W in place through lda
            W.p = a;
            W.rows = m;
            W.cols = n;
            W.ld = lda;
        } else {
            In A(C, loc, a, m, n, lda, "a");
            Wown = DMatBuf(C, m, n);
            copy_mat(C, A.m, Wown);
            W = Wown.m;
            sync(C);
        }
        Out Q(C, loc, q, m, cap, ldq, "q"), B(C, loc, b, cap, n, ldb, "b");
        QbOut r = qb_blocked(C, W, blk, num_blocks, tol, q_power, reorth_period, om, Q.m, B.m);
        if (Q.host && r.ell > 0) d2h_mat(C, Q.m.block(0, 0, m, r.ell), Q.host, Q.ldh);
        if (B.host && r.ell > 0) d2h_mat(C, B.m.block(0, 0, r.ell, n), B.host, B.ldh);
        if (loc == RLRA_HOST && inplace) d2h_mat(C, W, a, lda);
        sync(C);
        if (ell) *ell = r.ell;
        if (nhist) *nhist = int(r.hist.size());
        if (hist)
            for (size_t i = 0; i < r.hist.size(); ++i) hist[i] = r.hist[i];
        if (final_residual) *final_residual = r.final_residual;
        if (reached) *reached = r.reached ? 1 : 0;
    });
}

rlra_status rlra_svd_from_qb(rlra_ctx* ctx, int loc, const double* q, int m, int64_t ldq, const double* b,
                             int n, int64_t ldb, int ell, int k, int vnum, double* u, int64_t ldu,
                             double* sigma, double* v, int64_t ldv, int* k_out) {
    return guard(ctx, __func__, [&](Context& C) {
        if (k < 0 || k > ell) raise(RLRA_EDIM, fmt("rank k = %d outside [0, rank(B) = %d]", k, ell));
        if (k == 0) k = ell;
        if (k_out) *k_out = k;
        if (k == 0) return;
        In Q(C, loc, q, m, ell, ldq, "q"), B(C, loc, b, ell, n, ldb, "b");
        Out U(C, loc, u, m, k, ldu, "u"), V(C, loc, v, n, k, ldv, "v");
        OutVec<double> S(C, loc, sigma, k, "sigma");
        svd_from_qb(C, Q.m, B.m, k, vnum, U.m, S.d, V.m);
        U.finish(C);
        V.finish(C);
        S.finish(C);
        sync(C);
    });
}

rlra_status rlra_id_column(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda, int k,
                           double tol, int* jc, double* v, int64_t ldv, int* k_out, double* qr_residual,
                           int* reached, int* clamped) {
    return guard(ctx, __func__, [&](Context& C) {
        const int rmax = std::min(m, n);
        const bool tol_mode = (k == 0 && tol > 0.0);
        if (!tol_mode && (k < 1 || k > rmax || tol != 0.0))
            raise(RLRA_EDIM, fmt("pivoted_qr_partial: need either k in [1,%d] with tol=0 or k=0 with "
                                 "tol>0 (got k=%d, tol=%g)",
                                 rmax, k, tol));
        const int kmax = tol_mode ? rmax : k;
        In A(C, loc, a, m, n, lda, "a");
        OutVec<int> J(C, loc, jc, n, "jc");
        DMatBuf Vd(C, n, kmax);
        IdOut r = id_column(C, A.m, k, tol, J.d, Vd);
        Out V(C, loc, v, n, r.k, ldv, "v");
        if (r.k > 0) copy_mat(C, Vd.m.block(0, 0, n, r.k), V.m);
        V.finish(C);
        J.finish(C);
        sync(C);
        if (k_out) *k_out = r.k;
        if (qr_residual) *qr_residual = r.qr_residual;
        if (reached) *reached = r.reached ? 1 : 0;
        if (clamped) *clamped = r.clamped ? 1 : 0;
    });
}

rlra_status rlra_id_rand(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda, int k, int p,
                         int q, int s, const rlra_omega* omega, int* jc, double* v, int64_t ldv,
                         double* qr_residual, int* clamped) {
    return guard(ctx, __func__, [&](Context& C) {
        check_sample_rank(k, p, m, n);
        check_sample(k + p, q, s, n, m);
        OmegaSource om = omega_of(omega);
        In A(C, loc, a, m, n, lda, "a");
        OutVec<int> J(C, loc, jc, n, "jc");
        Out V(C, loc, v, n, k, ldv, "v");
        IdOut r = id_rand(C, A.m, k, p, q, s, om, J.d, V.m);
        V.finish(C);
        J.finish(C);
        sync(C);
        if (qr_residual) *qr_residual = r.qr_residual;
        if (clamped) *clamped = r.clamped ? 1 : 0;
    });
}

rlra_status rlra_two_sided_from_column(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda,
                                       const int* jc, int k, int* jr, double* w, int64_t ldw) {
    return guard(ctx, __func__, [&](Context& C) {
        if (k < 0 || k > std::min(m, n)) raise(RLRA_EDIM, fmt("two_sided_from_column: rank %d", k));
        OutVec<int> J(C, loc, jr, m, "jr");
        if (k == 0) {
            std::vector<int> id(m);
            for (int i = 0; i < m; ++i) id[i] = i;
            if (loc == RLRA_HOST)
                std::copy(id.begin(), id.end(), jr);
            else
                RLRA_CUDA(cudaMemcpyAsync(jr, id.data(), sizeof(int) * m, cudaMemcpyHostToDevice, C.stream));
            sync(C);
            return;
        }
        In A(C, loc, a, m, n, lda, "a");
        InVec<int> Jc(C, loc, jc, n, "jc");
        Out W(C, loc, w, m, k, ldw, "w");
        two_sided_from_column(C, A.m, Jc.d, k, J.d, W.m);
        W.finish(C);
        J.finish(C);
        sync(C);
    });
}

static void cur_core(Context& C, int loc, const DMat& A, const int* jc_d, const int* jr_d,
                     const DMat& V, int k, double* c, int64_t ldc, double* u, int64_t ldu, double* r,
                     int64_t ldr, double* residual) {
    const int m = int(A.rows), n = int(A.cols);
    if (k == 0) {
        if (residual) *residual = frobenius(C, A);
        return;
    }
    std::vector<int> jr_h(k);
    RLRA_CUDA(cudaMemcpyAsync(jr_h.data(), jr_d, sizeof(int) * k, cudaMemcpyDeviceToHost, C.stream));
    sync(C);
    Out Cm(C, loc, c, m, k, ldc, "c"), U(C, loc, u, k, k, ldu, "u"), R(C, loc, r, k, n, ldr, "r");
    const double res = cur_from_two_sided(C, A, jc_d, jr_d, V, k, Cm.m, U.m, R.m, jr_h.data());
    Cm.finish(C);
    U.finish(C);
    R.finish(C);
    sync(C);
    if (residual) *residual = res;
}

rlra_status rlra_cur_from_two_sided(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda,
                                    const int* jc, const int* jr, const double* v, int64_t ldv, int k,
                                    double* c, int64_t ldc, double* u, int64_t ldu, double* r,
                                    int64_t ldr, double* residual) {
    return guard(ctx, __func__, [&](Context& C) {
        In A(C, loc, a, m, n, lda, "a");
        InVec<int> Jc(C, loc, jc, n, "jc"), Jr(C, loc, jr, m, "jr");
        In V(C, loc, v, n, k, ldv, "v");
        cur_core(C, loc, A.m, Jc.d, Jr.d, V.m, k, c, ldc, u, ldu, r, ldr, residual);
    });
}

rlra_status rlra_cur_linkage(rlra_ctx* ctx, int loc, const double* r, int k, int n, int64_t ldr, const double* v,
                             int64_t ldv, const int* jr, double* u, int64_t ldu) {
    return guard(ctx, __func__, [&](Context& C) {
        if (k < 0 || n < 0) raise(RLRA_EDIM, fmt("cur_linkage: negative dimensions %dx%d", k, n));
        if (k == 0) return;
        if (n < k) raise(RLRA_EDIM, fmt("cur_linkage: R is %dx%d, need at least as many columns as rows", k, n));
        need(jr, "jr");
        In R(C, loc, r, k, n, ldr, "r"), V(C, loc, v, n, k, ldv, "v");
        Out U(C, loc, u, k, k, ldu, "u");
        cur_linkage(C, R.m, V.m, k, U.m, jr);
        U.finish(C);
        sync(C);
    });
}

rlra_status rlra_cur_rand(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda, int k, int p,
                          int q, int s, const rlra_omega* omega, int* jc, int* jr, double* v,
                          int64_t ldv, double* w, int64_t ldw, double* c, int64_t ldc, double* u,
                          int64_t ldu, double* r, int64_t ldr, double* residual, double* qr_residual) {
    return guard(ctx, __func__, [&](Context& C) {
        check_sample_rank(k, p, m, n);
        check_sample(k + p, q, s, n, m);
        OmegaSource om = omega_of(omega);
        In A(C, loc, a, m, n, lda, "a");
        OutVec<int> Jc(C, loc, jc, n, "jc"), Jr(C, loc, jr, m, "jr");
        Out V(C, loc, v, n, k, ldv, "v"), W(C, loc, w, m, k, ldw, "w");
        IdOut idr = id_rand(C, A.m, k, p, q, s, om, Jc.d, V.m);
        two_sided_from_column(C, A.m, Jc.d, k, Jr.d, W.m);
        cur_core(C, loc, A.m, Jc.d, Jr.d, V.m, k, c, ldc, u, ldu, r, ldr, residual);
        V.finish(C);
        W.finish(C);
        Jc.finish(C);
        Jr.finish(C);
        sync(C);
        if (qr_residual) *qr_residual = idr.qr_residual;
    });
}

}  // extern "C"
