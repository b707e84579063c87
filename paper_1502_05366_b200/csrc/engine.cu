// engine.cu — orchestration of the randomized factorizations on the device.
// Each function cites the reference lines whose semantics it restates; the
// arithmetic runs on the sm_100a kernels of gemm.cu, qr.cu, jacobi.cu and
// cpqr.cu.  Host code here only sequences launches and reads back the few
// scalars the reference's control flow branches on (the QB stop test, pivot
// and breakdown flags).
#include <chrono>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "cpqr.cuh"
#include "engine.cuh"
#include "hostio.cuh"
#include "gemm.cuh"
#include "jacobi.cuh"
#include "qr.cuh"
#include "reduce.cuh"

namespace rlra_b200 {

namespace {

__global__ void scale_cols_kernel(double* V, int64_t ldv, int n, int k, const double* sigma) {
    const int64_t tot = int64_t(n) * k;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e % n), j = int(e / n);
        V[i + int64_t(j) * ldv] *= 1.0 / sigma[j];
    }
}

__global__ void sqrt_vec_kernel(const double* d, int k, double* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x)
        out[i] = sqrt(d[i]);
}

__global__ void interp_kernel(const int* perm, const double* T, int64_t ldt, int n, int k, double* V,
                              int64_t ldv) {
    const int64_t tot = int64_t(n) * k;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int pos = int(e % n), j = int(e / n);
        const int row = perm[pos];
        double v;
        if (pos < k)
            v = (pos == j) ? 1.0 : 0.0;
        else
            v = T[j + int64_t(pos - k) * ldt];
        V[row + int64_t(j) * ldv] = v;
    }
}

int blocks_for(Context& ctx, int64_t total) {
    return int(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, int64_t(ctx.num_sms) * 8)));
}

double read_scalar(Context& ctx, const double* d) {
    RLRA_CUDA(cudaMemcpyAsync(ctx.h_scalars, d, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    return ctx.h_scalars[0];
}

// Philox Omega: materialised by philox_fill (n x l doubles — 82 MB at C5,
// 0.25% of A's bytes, 13 us of HBM writes) and multiplied by the plain GEMM,
// which streams A at the power-iteration GEMMs' rate; generating Omega inside
// the GEMM (GemmOpts::philox_b, the same bits) costs every M-tile the Philox
// work again and measured 7% slower at C5 (122.7 vs 114.8 ms).
// RLRA_SKETCH_FUSED=1 selects the in-GEMM generation.
bool sketch_fused() {
    static const bool v = [] {
        const char* e = std::getenv("RLRA_SKETCH_FUSED");
        return e && e[0] == '1';
    }();
    return v;
}

// Y = A * Omega_draw (op_a = N, Omega n x l) or Y = A^T * Omega_draw (op_a =
// T, Omega m x l).  Callback Omega is drawn on the host in the reference's
// order and uploaded.
}  // namespace

void sketch_philox(Context& ctx, Op op_a, int M, int l, int K, const double* A, int64_t lda, uint64_t seed, int draw,
                   int64_t krow0, double* Y, int64_t ldy) {
    if (sketch_fused()) {
        GemmOpts o;
        o.philox_b = true;
        o.seed = seed;
        o.draw = draw;
        o.krow0 = krow0;
        gemm(ctx, op_a, Op::N, M, l, K, 1.0, A, lda, nullptr, K, 0.0, Y, ldy, o);
        return;
    }
    DMatBuf Om(ctx, K, l);
    philox_fill(ctx, Om.m, seed, draw, krow0);
    gemm(ctx, op_a, Op::N, M, l, K, 1.0, A, lda, Om.m.p, Om.m.ld, 0.0, Y, ldy, GemmOpts{});
}

void sketch(Context& ctx, Op op_a, const DMat& A, int l, OmegaSource& om, const DMat& Y) {
    const int rows = int(op_a == Op::N ? A.cols : A.rows);
    const int draw = om.next_draw++;
    GemmTag tag(ctx, "gemm_sketch");
    if (om.o->mode == RLRA_OMEGA_PHILOX) {
        const int M = int(op_a == Op::N ? A.rows : A.cols);
        sketch_philox(ctx, op_a, M, l, rows, A.p, A.ld, om.o->seed, draw, 0, Y.p, Y.ld);
        return;
    }
    if (!om.o->fill) raise(RLRA_EINVAL, "rlra_omega: callback mode without a fill function");
    std::vector<double> h(size_t(rows) * l);
    om.o->fill(om.o->user, draw, rows, l, h.data());
    DMatBuf Om(ctx, rows, l);
    RLRA_CUDA(cudaMemcpyAsync(Om.m.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice,
                              ctx.stream));
    gemm(ctx, op_a, Op::N, 1.0, A, Om, 0.0, Y);
    // h must outlive the async copy
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
}

void orth(Context& ctx, const DMat& Y) { orth_inplace(ctx, Y, nullptr); }

// rsvd.hpp:144-156 finish_qb_qr_bt: Q m x l, Bt n x l (overwritten by Qhat)
void finish_qr_bt(Context& ctx, const DMat& Q, const DMat& Bt, int k, const DMat& U, double* sigma,
                  const DMat& V) {
    const int l = int(Bt.cols);
    DMatBuf R(ctx, l, l), Uh(ctx, l, l), Vh(ctx, l, l);
    Buf s(ctx, sizeof(double) * l);
    orth_inplace(ctx, Bt, &R.m);                       // compact_qr(bt)
    small_svd_tall(ctx, R, Uh, s.d(), Vh, true);       // small_svd(f.r)
    GemmTag tag(ctx, "gemm_lift");
    gemm(ctx, Op::N, Op::N, 1.0, Q, Vh.m.block(0, 0, l, k), 0.0, U);   // (Q*Vhat)(:,1:k)
    gemm(ctx, Op::N, Op::N, 1.0, Bt, Uh.m.block(0, 0, l, k), 0.0, V);  // (Qhat*Uhat)(:,1:k)
    RLRA_CUDA(cudaMemcpyAsync(sigma, s.p, sizeof(double) * k, cudaMemcpyDeviceToDevice, ctx.stream));
}

namespace {

// rsvd.hpp:115-140 finish_qb_bbt: Q m x l, B l x n
void finish_bbt(Context& ctx, const DMat& Q, const DMat& B, int k, const DMat& U, double* sigma,
                const DMat& V) {
    const int l = int(B.rows), n = int(B.cols);
    DMatBuf T(ctx, l, l), E(ctx, l, l);
    Buf d(ctx, sizeof(double) * l);
    gemm(ctx, Op::N, Op::T, 1.0, B, B, 0.0, T);  // B B^T
    sym_eig(ctx, T, d.d(), E);
    std::vector<double> hd(l);
    RLRA_CUDA(cudaMemcpyAsync(hd.data(), d.p, sizeof(double) * l, cudaMemcpyDeviceToHost, ctx.stream));
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    const double dmax = hd[0];
    for (int i = 0; i < k; ++i)
        if (hd[i] <= 0.0 || hd[i] < 1e-28 * dmax)
            raise(RLRA_ENUM, fmt("rank k exceeds numerical rank for v1; use v2 (eigenvalue %.3e at "
                                 "index %d vs max %.3e)",
                                 hd[i], i, dmax));
    sqrt_vec_kernel<<<1, 256, 0, ctx.stream>>>(d.d(), k, sigma);
    RLRA_LAUNCH_CHECK();
    ++ctx.launches;
    gemm(ctx, Op::N, Op::N, 1.0, Q, E.m.block(0, 0, l, k), 0.0, U);
    gemm(ctx, Op::T, Op::N, 1.0, B, E.m.block(0, 0, l, k), 0.0, V);
    scale_cols_kernel<<<blocks_for(ctx, int64_t(n) * k), 256, 0, ctx.stream>>>(V.p, V.ld, n, k, sigma);
    RLRA_LAUNCH_CHECK();
    ++ctx.launches;
}

}  // namespace

double frobenius(Context& ctx, const DMat& A) {
    Buf s(ctx, sizeof(double));
    sum_squares(ctx, A, s.d());
    return std::sqrt(read_scalar(ctx, s.d()));
}

void build_interp(Context& ctx, const int* perm, const DMat& T, int n, int k, const DMat& V) {
    if (k == 0) return;
    interp_kernel<<<blocks_for(ctx, int64_t(n) * k), 256, 0, ctx.stream>>>(perm, T.p, T.ld, n, k, V.p,
                                                                            V.ld);
    RLRA_LAUNCH_CHECK();
    ++ctx.launches;
}

// Re-orthonormalisation between half-multiplies.  Every such basis is
// consumed only through its span by the next product, so span_only callers
// (rsvd, id_rand: the sample is never returned) use one CholQR pass; the
// public sample_right/left keep the reference's fully orthonormal iterates.
static void orth_mid(Context& ctx, const DMat& Y, bool span_only) {
    if (span_only)
        orth_span_inplace(ctx, Y);
    else
        orth_inplace(ctx, Y, nullptr);
}

void sample_right(Context& ctx, const DMat& A, int l, int q, int s, OmegaSource& om, const DMat& Y,
                  bool span_only, bool sketched, const DMat* zpre) {
    const int n = int(A.cols);
    if (!sketched) sketch(ctx, Op::N, A, l, om, Y);  // Y = A * Omega
    if (q == 0) return;
    DMatBuf Z(ctx, n, l), Y2;
    if (span_only) Y2 = DMatBuf(ctx, Y.rows, l);  // span-only orth output: no copy back into Y
    GemmTag tag(ctx, "gemm_power");
    for (int j = 1; j <= q; ++j) {
        if (j == 1 && zpre && span_only) {
            // A^T Q = (A^T Y) R^{-1} with Y = Q R the CholQR pass sketch.hpp:54
            // asks for: the span the reference's orth(Y) then A^T Q produce,
            // without streaming A a second time (A^T Y was summed under the
            // upload).  Rounding differs from A^T (Y R^{-1}) by ~u kappa(Y).
            // Only for a well-conditioned Y (every Cholesky pivot >= 1e-8 of its
            // diagonal, i.e. kappa(Y) below ~1e4): the reordering costs
            // ~u kappa(Y) in Z, kept at the 1e-12 level (C5: sigma within
            // 2.4e-14 of the device-resident order).
            DMatBuf Ri(ctx, l, l);
            if (span_rinv(ctx, Y, Ri.m, 1e-8)) {
                GemmOpts tri;
                tri.tri_b_upper = true;
                gemm(ctx, Op::N, Op::N, 1.0, *zpre, Ri.m, 0.0, Z.m, tri);
                if ((2 * j - 1) % s == 0) orth_mid(ctx, Z, span_only);
                gemm(ctx, Op::N, Op::N, 1.0, A, Z, 0.0, Y);  // Y = A Z
                continue;
            }
            // too ill-conditioned for one CholQR pass: the standard step below
        }
        DMat Yc = Y;
        if ((2 * j - 2) % s == 0) {
            if (span_only && orth_span_into(ctx, Y, Y2.m))
                Yc = Y2.m;
            else
                orth_mid(ctx, Y, span_only);
        }
        gemm(ctx, Op::T, Op::N, 1.0, A, Yc, 0.0, Z);  // Z = A^T Y
        if ((2 * j - 1) % s == 0) orth_mid(ctx, Z, span_only);
        gemm(ctx, Op::N, Op::N, 1.0, A, Z, 0.0, Y);  // Y = A Z
    }
}

void sample_left_t(Context& ctx, const DMat& A, int l, int q, int s, OmegaSource& om, const DMat& Yt,
                   bool span_only) {
    const int m = int(A.rows);
    sketch(ctx, Op::T, A, l, om, Yt);  // (A^T) * Omega~, Omega~ m x l
    if (q == 0) return;
    DMatBuf Z(ctx, m, l);
    GemmTag tag(ctx, "gemm_power");
    for (int j = 1; j <= q; ++j) {
        if ((2 * j - 2) % s == 0) orth_mid(ctx, Yt, span_only);
        gemm(ctx, Op::N, Op::N, 1.0, A, Yt, 0.0, Z);  // (A^T)^T Yt
        if ((2 * j - 1) % s == 0) orth_mid(ctx, Z, span_only);
        gemm(ctx, Op::T, Op::N, 1.0, A, Z, 0.0, Yt);
    }
}

bool upload_and_sketch(Context& ctx, const double* hA, int64_t lda, const DMat& dA, int l, OmegaSource& om,
                       const DMat& Y, const DMat* Zt) {
    const int64_t m = dA.rows, n = dA.cols;
    if (m <= 0 || n <= 0) {
        // an empty row shard still consumes its Omega draw (callback mode: the
        // caller's RngState advances exactly as on the other ranks)
        const int draw = om.next_draw++;
        if (om.o->mode != RLRA_OMEGA_PHILOX && om.o->fill && n > 0) {
            std::vector<double> h(size_t(n) * l);
            om.o->fill(om.o->user, draw, int(n), l, h.data());
        }
        if (Zt) zero_mat(ctx, *Zt);
        return Zt != nullptr;
    }
    if (!ctx.copy_stream) RLRA_CUDA(cudaStreamCreateWithFlags(&ctx.copy_stream, cudaStreamNonBlocking));
    // Omega once (callback mode: the reference's draw, uploaded; Philox: philox_fill)
    const int draw = om.next_draw++;
    DMatBuf Om;
    std::vector<double> h;
    const bool fused = om.o->mode == RLRA_OMEGA_PHILOX && sketch_fused();
    if (om.o->mode == RLRA_OMEGA_PHILOX && !fused) {
        Om = DMatBuf(ctx, n, l);
        philox_fill(ctx, Om.m, om.o->seed, draw, 0);
    } else if (om.o->mode != RLRA_OMEGA_PHILOX) {
        if (!om.o->fill) raise(RLRA_EINVAL, "rlra_omega: callback mode without a fill function");
        h.resize(size_t(n) * l);
        om.o->fill(om.o->user, draw, int(n), l, h.data());
        Om = DMatBuf(ctx, n, l);
        RLRA_CUDA(cudaMemcpyAsync(Om.m.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice,
                                  ctx.stream));
    }
    const auto t_up0 = std::chrono::steady_clock::now();
    // row chunks of whole 128-row GEMM tiles, ~32 of them for a large A (the
    // last chunk's sketch is the only part not hidden under the upload)
    const int64_t bytes = m * n * 8;
    const int64_t nchunk = bytes >= (int64_t(256) << 20) ? 32 : 1;
    const int64_t rows = std::max<int64_t>(128, ((m + nchunk - 1) / nchunk + 127) / 128 * 128);
    std::vector<cudaEvent_t> ev;
    cudaEvent_t ready;
    RLRA_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    RLRA_CUDA(cudaEventRecord(ready, ctx.stream));  // dA / Y / Omega allocations are stream-ordered
    RLRA_CUDA(cudaStreamWaitEvent(ctx.copy_stream, ready, 0));
    GemmTag tag(ctx, "gemm_sketch");
    for (int64_t r0 = 0; r0 < m; r0 += rows) {
        const int64_t nr = std::min(rows, m - r0);
        h2d_copy(ctx, ctx.copy_stream, hA + r0, lda, dA.block(r0, 0, nr, n));  // pageable: staged
        cudaEvent_t e;
        RLRA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        RLRA_CUDA(cudaEventRecord(e, ctx.copy_stream));
        ev.push_back(e);
        RLRA_CUDA(cudaStreamWaitEvent(ctx.stream, e, 0));
        const DMat Ar = dA.block(r0, 0, nr, n), Yr = Y.block(r0, 0, nr, l);
        if (fused) {
            GemmOpts o;
            o.philox_b = true;
            o.seed = om.o->seed;
            o.draw = draw;
            gemm(ctx, Op::N, Op::N, int(nr), l, int(n), 1.0, Ar.p, Ar.ld, nullptr, n, 0.0, Yr.p, Yr.ld, o);
        } else {
            gemm(ctx, Op::N, Op::N, 1.0, Ar, Om.m, 0.0, Yr);
        }
        if (Zt && nchunk > 1) {  // Zt += A_c^T Y_c, chunks summed in order (deterministic)
            GemmTag zt(ctx, "gemm_power");
            gemm(ctx, Op::T, Op::N, 1.0, Ar, Yr, r0 == 0 ? 0.0 : 1.0, *Zt);
        }
    }
    static const bool times = std::getenv("RLRA_HOSTIO_TIMES") != nullptr;
    const auto t_enq = std::chrono::steady_clock::now();
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));  // h (callback Omega) outlives its copy; events done
    if (times)
        std::fprintf(stderr, "upload_and_sketch %lld x %lld: enqueued %.3f ms, done %.3f ms\n", (long long)m,
                     (long long)n, std::chrono::duration<double, std::milli>(t_enq - t_up0).count(),
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_up0).count());
    for (auto e : ev) cudaEventDestroy(e);
    cudaEventDestroy(ready);
    return Zt && nchunk > 1;
}

void rsvd(Context& ctx, int variant, const DMat& A, int k, int p, int q, int s, OmegaSource& om,
          const DMat& U, double* sigma, const DMat& V, const DMat* sketched, const DMat* zpre) {
    const int m = int(A.rows), n = int(A.cols), l = k + p;
    DMatBuf Yown;
    DMat Y;
    if (sketched) {
        Y = *sketched;
    } else {
        Yown = DMatBuf(ctx, m, l);
        Y = Yown.m;
    }
    if (variant == RLRA_RSVD_BASIC) {
        // rsvd.hpp:127-140 (Fig. 1): Y = A G, Q = orth(Y), B = Q^T A, small_svd(B)
        if (!sketched) sketch(ctx, Op::N, A, l, om, Y);
        orth(ctx, Y);
        DMatBuf B(ctx, l, n);
        gemm(ctx, Op::T, Op::N, 1.0, Y, A, 0.0, B);
        const int r = std::min(l, n);
        DMatBuf Ub(ctx, l, r), Vb(ctx, n, r);
        Buf sb(ctx, sizeof(double) * r);
        small_svd(ctx, B, Ub, sb.d(), Vb);
        gemm(ctx, Op::N, Op::N, 1.0, Y, Ub.m.block(0, 0, l, k), 0.0, U);
        copy_mat(ctx, Vb.m.block(0, 0, n, k), V);
        RLRA_CUDA(cudaMemcpyAsync(sigma, sb.p, sizeof(double) * k, cudaMemcpyDeviceToDevice, ctx.stream));
        return;
    }
    sample_right(ctx, A, l, q, s, om, Y, /*span_only=*/true, /*sketched=*/sketched != nullptr, zpre);
    orth(ctx, Y);
    GemmTag tag(ctx, "gemm_proj");
    if (variant == RLRA_RSVD_V2) {
        DMatBuf Bt(ctx, n, l);
        gemm(ctx, Op::T, Op::N, 1.0, A, Y, 0.0, Bt);  // Bt = A^T Q (rsvd.hpp:158)
        finish_qr_bt(ctx, Y, Bt, k, U, sigma, V);
    } else {
        DMatBuf B(ctx, l, n);
        gemm(ctx, Op::T, Op::N, 1.0, Y, A, 0.0, B);  // B = Q^T A (rsvd.hpp:148)
        finish_bbt(ctx, Y, B, k, U, sigma, V);
    }
}

QbOut qb_blocked(Context& ctx, const DMat& W, int blk, int num_blocks, double tol, int q_power,
                 int reorth_period, OmegaSource& om, const DMat& Q, const DMat& B) {
    const int m = int(W.rows), n = int(W.cols), rmax = std::min(m, n);
    QbOut out;
    Buf sq(ctx, sizeof(double));
    double resid = frobenius(ctx, W);
    DMatBuf Z(ctx, n, blk), P(ctx, std::max(1, int(Q.cols)), blk);
    for (int i = 1; i <= num_blocks; ++i) {
        const int width = std::min(blk, rmax - out.ell);
        if (width < 1) break;
        const DMat Qi = Q.block(0, out.ell, m, width);
        const DMat Zi = Z.m.block(0, 0, n, width);
        // Q_i must leave this block orthonormal; every earlier orth only feeds
        // the span of the next product (or of the reorth projection).
        const bool reorth = (i % reorth_period == 0);
        sketch(ctx, Op::N, W, width, om, Qi);  // W * Omega_i (qb.hpp:119-121)
        orth_mid(ctx, Qi, q_power > 0 || reorth);
        for (int j = 0; j < q_power; ++j) {
            gemm(ctx, Op::T, Op::N, 1.0, W, Qi, 0.0, Zi);
            orth_mid(ctx, Zi, true);
            gemm(ctx, Op::N, Op::N, 1.0, W, Zi, 0.0, Qi);
            orth_mid(ctx, Qi, j + 1 < q_power || reorth);
        }
        if (reorth) {  // qb.hpp:126-130
            if (out.ell > 0) {
                const DMat Qp = Q.block(0, 0, m, out.ell);
                const DMat Pi = P.m.block(0, 0, out.ell, width);
                gemm(ctx, Op::T, Op::N, 1.0, Qp, Qi, 0.0, Pi);
                gemm(ctx, Op::N, Op::N, -1.0, Qp, Pi, 1.0, Qi);
            }
            orth(ctx, Qi);
        }
        const DMat Bi = B.block(out.ell, 0, width, n);
        gemm(ctx, Op::T, Op::N, 1.0, Qi, W, 0.0, Bi);  // B_i = Q_i^T W
        // W <- W - Q_i B_i and ||W||_F^2 in one pass (qb.hpp:135-137)
        GemmOpts o;
        o.epi = EPI_RESID;
        o.R = W.p;
        o.ldr = W.ld;
        o.resid_sq = sq.d();
        gemm(ctx, Op::N, Op::N, m, n, width, 1.0, Qi.p, Qi.ld, Bi.p, Bi.ld, 0.0, W.p, W.ld, o);
        out.ell += width;
        resid = std::sqrt(read_scalar(ctx, sq.d()));
        out.hist.push_back(resid);
        if (tol > 0.0 && resid < tol) {
            out.final_residual = resid;
            out.reached = true;
            return out;
        }
    }
    out.final_residual = resid;
    out.reached = !(tol > 0.0);
    return out;
}

// ||A - Q B||_F through the fused residual GEMM (A copied: the epilogue is
// read-only on R when C is null)
static double qb_residual(Context& ctx, const DMat& A, const DMat& Q, const DMat& B) {
    Buf sq(ctx, sizeof(double));
    GemmOpts o;
    o.epi = EPI_RESID;
    o.R = A.p;
    o.ldr = A.ld;
    o.resid_sq = sq.d();
    gemm(ctx, Op::N, Op::N, int(A.rows), int(A.cols), int(Q.cols), 1.0, Q.p, Q.ld, B.p, B.ld, 0.0, nullptr, 0, o);
    return std::sqrt(read_scalar(ctx, sq.d()));
}

double qb_parallel(Context& ctx, const DMat& A, int blk, int num_blocks, int q_power, OmegaSource& om, const DMat& Q,
                   const DMat& B) {
    const int m = int(A.rows), n = int(A.cols);
    DMatBuf Y(ctx, m, blk), Z(ctx, n, blk), P(ctx, blk * num_blocks, blk);
    for (int i = 0; i < num_blocks; ++i) {  // qb.hpp:176-186, node i draws its block directly
        const DMat Qi = Q.block(0, int64_t(i) * blk, m, blk);
        OmegaSource oi{om.o, i << 16};
        sketch(ctx, Op::N, A, blk, oi, Qi);  // y_i = A Omega_i
        for (int j = 0; j < q_power; ++j) {
            orth(ctx, Qi);
            gemm(ctx, Op::T, Op::N, 1.0, A, Qi, 0.0, Z.m);
            orth(ctx, Z.m);
            gemm(ctx, Op::N, Op::N, 1.0, A, Z.m, 0.0, Qi);
        }
        orth(ctx, Qi);  // qb.hpp:188-189
    }
    for (int i = 1; i < num_blocks; ++i) {  // qb.hpp:191-198: sequential projection
        const DMat Qp = Q.block(0, 0, m, int64_t(i) * blk), Qi = Q.block(0, int64_t(i) * blk, m, blk);
        const DMat Pi = P.m.block(0, 0, int64_t(i) * blk, blk);
        gemm(ctx, Op::T, Op::N, 1.0, Qp, Qi, 0.0, Pi);
        gemm(ctx, Op::N, Op::N, -1.0, Qp, Pi, 1.0, Qi);
        orth(ctx, Qi);
    }
    gemm(ctx, Op::T, Op::N, 1.0, Q, A, 0.0, B);  // B = Q^T A
    return qb_residual(ctx, A, Q, B);
}

double qb_hierarchical(Context& ctx, const DMat& A, int num_row_blocks, int blk, int num_blocks, int q_power,
                       OmegaSource& om, const DMat& Q, const DMat& B) {
    const int m = int(A.rows), n = int(A.cols), blocks = num_row_blocks, rank = blk * num_blocks;
    const int base = m / blocks;
    struct Node {
        DMatBuf q, b;
        int row0 = 0, rows = 0;
    };
    std::vector<Node> nodes(static_cast<size_t>(blocks));
    int row0 = 0;
    for (int t = 0; t < blocks; ++t) {  // leaves (qb.hpp:235-244), node t's substreams
        const int rows_t = (t == blocks - 1) ? m - row0 : base;
        DMatBuf W(ctx, rows_t, n);
        copy_mat(ctx, A.block(row0, 0, rows_t, n), W.m);
        nodes[size_t(t)].q = DMatBuf(ctx, rows_t, rank);
        nodes[size_t(t)].b = DMatBuf(ctx, rank, n);
        nodes[size_t(t)].row0 = row0;
        nodes[size_t(t)].rows = rows_t;
        OmegaSource ot{om.o, t << 16};
        qb_blocked(ctx, W.m, blk, num_blocks, 0.0, q_power, 1, ot, nodes[size_t(t)].q.m, nodes[size_t(t)].b.m);
        row0 += rows_t;
    }
    int merge = blocks;  // merge nodes follow the leaves (qb.hpp:245-263)
    while (nodes.size() > 1) {
        std::vector<Node> next;
        for (size_t t = 0; t + 1 < nodes.size(); t += 2) {
            Node& L = nodes[t];
            Node& Rn = nodes[t + 1];
            DMatBuf S(ctx, 2 * rank, n), Qm(ctx, 2 * rank, rank);
            copy_mat(ctx, L.b.m, S.m.block(0, 0, rank, n));
            copy_mat(ctx, Rn.b.m, S.m.block(rank, 0, rank, n));
            Node M;
            M.b = DMatBuf(ctx, rank, n);
            OmegaSource omg{om.o, (merge++) << 16};
            qb_blocked(ctx, S.m, blk, num_blocks, 0.0, q_power, 1, omg, Qm.m, M.b.m);
            M.row0 = L.row0;
            M.rows = L.rows + Rn.rows;
            M.q = DMatBuf(ctx, M.rows, rank);
            gemm(ctx, Op::N, Op::N, 1.0, L.q.m, Qm.m.block(0, 0, rank, rank), 0.0, M.q.m.block(0, 0, L.rows, rank));
            gemm(ctx, Op::N, Op::N, 1.0, Rn.q.m, Qm.m.block(rank, 0, rank, rank), 0.0,
                 M.q.m.block(L.rows, 0, Rn.rows, rank));
            next.push_back(std::move(M));
        }
        nodes = std::move(next);
    }
    copy_mat(ctx, nodes[0].q.m, Q);
    copy_mat(ctx, nodes[0].b.m, B);
    return qb_residual(ctx, A, Q, B);
}

void svd_from_qb(Context& ctx, const DMat& Q, const DMat& B, int k, int vnum, const DMat& U,
                 double* sigma, const DMat& V) {
    const int ell = int(B.rows), n = int(B.cols);
    if (vnum == RLRA_VNUM_BBT) return finish_bbt(ctx, Q, B, k, U, sigma, V);
    DMatBuf Bt(ctx, n, ell);
    transpose_mat(ctx, B, Bt);
    finish_qr_bt(ctx, Q, Bt, k, U, sigma, V);
}

IdOut id_column(Context& ctx, const DMat& A, int k, double tol, int* jc, const DMat& V) {
    const int m = int(A.rows), n = int(A.cols);
    const int rmax = std::min(m, n);
    const bool tol_mode = (k == 0 && tol > 0.0);
    const int kmax = tol_mode ? rmax : std::max(k, 1);
    DMatBuf S1(ctx, kmax, n);
    CpqrResult r = pivoted_qr(ctx, A, k, tol, nullptr, S1, jc);
    IdOut out;
    out.k = r.frank;
    out.qr_residual = r.residual;
    out.reached = tol > 0.0 ? r.reached : true;
    const int f = r.frank;
    if (f == 0) return out;
    DMatBuf T(ctx, f, std::max(1, n - f));
    if (n > f)
        out.clamped = upper_tri_solve(ctx, S1.m.block(0, 0, f, f), S1.m.block(0, f, f, n - f),
                                      T.m.block(0, 0, f, n - f));
    build_interp(ctx, jc, T, n, f, V);
    return out;
}

IdOut id_rand(Context& ctx, const DMat& A, int k, int p, int q, int s, OmegaSource& om, int* jc,
              const DMat& V) {
    const int n = int(A.cols), l = k + p;
    DMatBuf Yt(ctx, n, l), Y(ctx, l, n), S1(ctx, l, n);
    sample_left_t(ctx, A, l, q, s, om, Yt, /*span_only=*/true);
    transpose_mat(ctx, Yt, Y);
    pivoted_qr(ctx, Y, l, 0.0, nullptr, S1, jc);  // interp.hpp:209
    IdOut out;
    out.k = k;
    {
        Buf sq(ctx, sizeof(double));
        sum_squares(ctx, S1.m.block(k, k, l - k, n - k), sq.d());  // interp.hpp:213
        out.qr_residual = std::sqrt(read_scalar(ctx, sq.d()));
    }
    DMatBuf T(ctx, k, std::max(1, n - k));
    if (n > k)
        out.clamped = upper_tri_solve(ctx, S1.m.block(0, 0, k, k), S1.m.block(0, k, k, n - k),
                                      T.m.block(0, 0, k, n - k));
    build_interp(ctx, jc, T, n, k, V);
    return out;
}

void two_sided_from_column(Context& ctx, const DMat& A, const int* jc, int k, int* jr, const DMat& Wr) {
    const int m = int(A.rows);
    DMatBuf C(ctx, m, k), Ct(ctx, k, m);
    gather_cols(ctx, A, jc, k, C);
    transpose_mat(ctx, C, Ct);
    id_column(ctx, Ct, k, 0.0, jr, Wr);  // id_row(c, k) = id_column(c^T, k)
}

// cur_linkage (interp.hpp:143-156): U = argmin ||U R - V^T||_F via
// compact_qr(R^T), the skeleton-row rank check, and a triangular solve
void cur_linkage(Context& ctx, const DMat& R, const DMat& V, int k, const DMat& U, const int* jr_host) {
    const int n = int(R.cols);
    DMatBuf Rt(ctx, n, k), Rh(ctx, k, k), X(ctx, k, k), T(ctx, k, k);
    transpose_mat(ctx, R, Rt);
    orth_inplace(ctx, Rt, &Rh.m);
    {
        std::vector<double> h(size_t(k) * k);
        RLRA_CUDA(cudaMemcpyAsync(h.data(), Rh.m.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost,
                                  ctx.stream));
        RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
        double dmax = 0.0;
        for (int i = 0; i < k; ++i) dmax = std::max(dmax, std::fabs(h[i + size_t(i) * k]));
        for (int i = 0; i < k; ++i)
            if (dmax == 0.0 || std::fabs(h[i + size_t(i) * k]) < 1e-13 * dmax)
                raise(RLRA_ENUM, fmt("CUR linkage: skeleton row %d makes R rank-deficient to working "
                                     "precision",
                                     jr_host[i]));
    }
    gemm(ctx, Op::T, Op::N, 1.0, Rt, V, 0.0, X);  // Qhat^T V
    upper_tri_solve(ctx, Rh, X, T);
    transpose_mat(ctx, T, U);
}

double cur_from_two_sided(Context& ctx, const DMat& A, const int* jc, const int* jr, const DMat& V,
                          int k, const DMat& C, const DMat& U, const DMat& R, const int* jr_host) {
    const int m = int(A.rows), n = int(A.cols);
    gather_cols(ctx, A, jc, k, C);
    gather_rows(ctx, A, jr, k, R);
    cur_linkage(ctx, R, V, k, U, jr_host);
    // ||A - C (U R)||_F, fused GEMM + subtract + sum of squares (K10)
    DMatBuf UR(ctx, k, n);
    gemm(ctx, Op::N, Op::N, 1.0, U, R, 0.0, UR);
    Buf sq(ctx, sizeof(double));
    GemmOpts o;
    o.epi = EPI_RESID;
    o.R = A.p;
    o.ldr = A.ld;
    o.resid_sq = sq.d();
    gemm(ctx, Op::N, Op::N, m, n, k, 1.0, C.p, C.ld, UR.m.p, UR.m.ld, 0.0, nullptr, 0, o);
    return std::sqrt(read_scalar(ctx, sq.d()));
}

}  // namespace rlra_b200
