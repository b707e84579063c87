// io.cu — the components either side of the path:
//   * binary matrix I/O straight to (or from) device row shards, in the
//     reference's format and with its validator and messages (io.hpp:40-109):
//     8-byte header (int32 rows, cols, little-endian) + rows*cols doubles in
//     row order; the file is exactly 8 + 8*rows*cols bytes; every value must
//     be finite.  The loader streams row chunks through two pinned buffers,
//     transposes them on the GPU into the column-major shard and checks
//     finiteness there (first offending element reported like the reference);
//   * the test-matrix generator (testmat.hpp:65-74 semantics: A = U diag(s)
//     V^T + noise G with U, V orthonormalised Gaussians; Philox draws);
//   * the SVD verifier (report.hpp:97-138: relative Frobenius error, the
//     60-step power-iteration spectral estimate of norms.hpp:41-56 with the
//     reference's fixed RngState 0x5bd1e995 start vectors, and the floors).
#include <cstdio>
#include <cstring>

#include "engine.cuh"
#include "gemm.cuh"
#include "io.cuh"
#include "dist.cuh"
#include "qr.cuh"
#include "reduce.cuh"

namespace rlra_b200 {

namespace {

// row-major chunk (rows x n, contiguous) -> column-major dst rows [r0, r0+rows)
// and the smallest global linear index (row * n + col) of a non-finite value
__global__ void rowmajor_to_colmajor_kernel(const double* src, int rows, int n, double* dst, int64_t ldd,
                                            int64_t grow0, unsigned long long* first_bad) {
    const int64_t tot = int64_t(rows) * n;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e / n), j = int(e % n);
        const double v = src[e];
        dst[i + int64_t(j) * ldd] = v;
        if (!isfinite(v)) atomicMin(first_bad, (unsigned long long)((grow0 + i) * int64_t(n) + j));
    }
}

__global__ void colmajor_to_rowmajor_kernel(const double* src, int64_t lds, int rows, int n, double* dst) {
    const int64_t tot = int64_t(rows) * n;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e / n), j = int(e % n);
        dst[e] = src[i + int64_t(j) * lds];
    }
}

__global__ void scale_cols_by_kernel(double* X, int64_t ldx, int rows, int cols, const double* s) {
    const int64_t tot = int64_t(rows) * cols;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e % rows), j = int(e / rows);
        X[i + int64_t(j) * ldx] *= s[j];
    }
}

__global__ void axpy_mat_kernel(double* Y, int64_t ldy, const double* X, int64_t ldx, int rows, int cols,
                                double alpha) {
    const int64_t tot = int64_t(rows) * cols;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e % rows), j = int(e / rows);
        Y[i + int64_t(j) * ldy] += alpha * X[i + int64_t(j) * ldx];
    }
}

// y = A x (A m x n column-major): one thread per row, columns streamed
__global__ void gemv_n_kernel(const double* A, int64_t lda, int m, int n, const double* x, double* y) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += A[i + int64_t(j) * lda] * x[j];
        y[i] = s;
    }
}

// y = A^T x: one warp per column
__global__ void gemv_t_kernel(const double* A, int64_t lda, int m, int n, const double* x, double* y) {
    const int lane = threadIdx.x & 31;
    for (int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n; j += (gridDim.x * blockDim.x) >> 5) {
        double s = 0.0;
        for (int i = lane; i < m; i += 32) s += A[i + int64_t(j) * lda] * x[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) y[j] = s;
    }
}

__global__ void scale_vec_kernel(double* v, int n, const double* nrm2) {
    const double inv = 1.0 / sqrt(*nrm2);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] *= inv;
}

int grid_for(Context& ctx, int64_t work) {
    return int(std::max<int64_t>(1, std::min<int64_t>(int64_t(ctx.num_sms) * 8, (work + 255) / 256)));
}

void gemv(Context& ctx, bool trans, const DMat& A, const double* x, double* y) {
    if (!trans)
        gemv_n_kernel<<<grid_for(ctx, A.rows), 256, 0, ctx.stream>>>(A.p, A.ld, int(A.rows), int(A.cols), x, y);
    else
        gemv_t_kernel<<<grid_for(ctx, A.cols * 32), 256, 0, ctx.stream>>>(A.p, A.ld, int(A.rows), int(A.cols), x, y);
    RLRA_LAUNCH_CHECK();
    ++ctx.launches;
}

double sq_norm(Context& ctx, const double* v, int n, double* scratch) {
    DMat d;
    d.p = const_cast<double*>(v);
    d.rows = n;
    d.cols = 1;
    d.ld = std::max(n, 1);
    sum_squares(ctx, d, scratch);
    RLRA_CUDA(cudaMemcpyAsync(ctx.h_scalars, scratch, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    return ctx.h_scalars[0];
}

// spectral_norm_est (norms.hpp:41-56) of A - X Y^T (X, Y may be empty):
// v from the host RngState, 60 power steps
double spectral_est(Context& ctx, const DMat& A, const DMat* X, const DMat* Y, int iters, rlra_rng* rng) {
    const int m = int(A.rows), n = int(A.cols);
    if (m == 0 || n == 0) return 0.0;
    std::vector<double> hv(n);
    rlra_rng_gaussian_fill(rng, n, 1, hv.data());
    Buf v(ctx, sizeof(double) * n), w(ctx, sizeof(double) * m), t(ctx, sizeof(double) * std::max<int64_t>(1, X ? X->cols : 1)),
        sc(ctx, sizeof(double) * 2);
    RLRA_CUDA(cudaMemcpyAsync(v.p, hv.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx.stream));
    const int k = X ? int(X->cols) : 0;
    double sigma = 0.0;
    for (int it = 0; it < iters; ++it) {
        const double vn2 = sq_norm(ctx, v.d(), n, sc.d());
        if (vn2 == 0.0) return 0.0;
        scale_vec_kernel<<<grid_for(ctx, n), 256, 0, ctx.stream>>>(v.d(), n, sc.d());
        RLRA_LAUNCH_CHECK();
        gemv(ctx, false, A, v.d(), w.d());  // w = A v
        if (k > 0) {                          //   - X (Y^T v)
            gemv(ctx, true, *Y, v.d(), t.d());
            Buf xt(ctx, sizeof(double) * m);
            gemv(ctx, false, *X, t.d(), xt.d());
            axpy_mat_kernel<<<grid_for(ctx, m), 256, 0, ctx.stream>>>(w.d(), m, xt.d(), m, m, 1, -1.0);
            RLRA_LAUNCH_CHECK();
        }
        sigma = std::sqrt(sq_norm(ctx, w.d(), m, sc.d()));
        gemv(ctx, true, A, w.d(), v.d());  // v = A^T w
        if (k > 0) {                         //   - Y (X^T w)
            gemv(ctx, true, *X, w.d(), t.d());
            Buf yt(ctx, sizeof(double) * n);
            gemv(ctx, false, *Y, t.d(), yt.d());
            axpy_mat_kernel<<<grid_for(ctx, n), 256, 0, ctx.stream>>>(v.d(), n, yt.d(), n, n, 1, -1.0);
            RLRA_LAUNCH_CHECK();
        }
    }
    return sigma;
}

struct File {
    FILE* f = nullptr;
    explicit File(const std::string& path, const char* mode) : f(std::fopen(path.c_str(), mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

void put_i32_le(unsigned char* p, int32_t v) {
    const uint32_t u = uint32_t(v);
    for (int i = 0; i < 4; ++i) p[i] = (unsigned char)((u >> (8 * i)) & 0xff);
}
int32_t get_i32_le(const unsigned char* p) {
    uint32_t u = 0;
    for (int i = 0; i < 4; ++i) u |= uint32_t(p[i]) << (8 * i);
    return int32_t(u);
}

}  // namespace

BinaryHeader read_binary_header(const std::string& path) {
    File fl(path, "rb");
    if (!fl.f) raise(RLRA_EIO, fmt("load_binary: cannot open '%s'", path.c_str()));
    std::fseek(fl.f, 0, SEEK_END);
    const long long size = std::ftell(fl.f);
    std::fseek(fl.f, 0, SEEK_SET);
    if (size < 8)
        raise(RLRA_EIO, fmt("load_binary: '%s' truncated at byte offset %lld: need 8 header bytes", path.c_str(), size));
    unsigned char hdr[8];
    if (std::fread(hdr, 1, 8, fl.f) != 8) raise(RLRA_EIO, fmt("load_binary: read from '%s' failed at byte offset 0", path.c_str()));
    BinaryHeader h;
    h.rows = get_i32_le(hdr);
    h.cols = get_i32_le(hdr + 4);
    if (h.rows <= 0 || h.cols <= 0)
        raise(RLRA_EIO, fmt("load_binary: '%s' has invalid dimensions %d x %d in header at byte offset 0", path.c_str(),
                            h.rows, h.cols));
    const long long expected = 8LL + 8LL * h.rows * h.cols;
    if (size < expected)
        raise(RLRA_EIO, fmt("load_binary: '%s' truncated at byte offset %lld: %d x %d payload needs %lld bytes",
                            path.c_str(), size, h.rows, h.cols, expected));
    if (size > expected)
        raise(RLRA_EIO, fmt("load_binary: '%s' is %lld bytes but a %d x %d matrix occupies exactly %lld",
                            path.c_str(), size, h.rows, h.cols, expected));
    return h;
}

void load_binary_rows(Context& ctx, const std::string& path, int64_t row0, const DMat& dst) {
    const BinaryHeader h = read_binary_header(path);
    const int n = h.cols;
    const int64_t rows = dst.rows;
    if (dst.cols != n || row0 < 0 || row0 + rows > h.rows)
        raise(RLRA_EDIM, fmt("load_binary: rows [%lld, %lld) x %d requested from a %d x %d file", (long long)row0,
                             (long long)(row0 + rows), int(dst.cols), h.rows, h.cols));
    if (rows == 0) return;
    File fl(path, "rb");
    if (!fl.f) raise(RLRA_EIO, fmt("load_binary: cannot open '%s'", path.c_str()));
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t(64) << 20) / (8LL * n)));
    double* pin[2] = {nullptr, nullptr};
    cudaEvent_t ev[2];
    Buf stage[2] = {Buf(ctx, sizeof(double) * size_t(chunk) * n), Buf(ctx, sizeof(double) * size_t(chunk) * n)};
    Buf bad(ctx, sizeof(unsigned long long));
    RLRA_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), ctx.stream));
    for (int b = 0; b < 2; ++b) {
        RLRA_CUDA(cudaMallocHost(&pin[b], sizeof(double) * size_t(chunk) * n));
        RLRA_CUDA(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
    }
    struct Cleanup {
        double** pin;
        cudaEvent_t* ev;
        ~Cleanup() {
            for (int b = 0; b < 2; ++b) {
                if (pin[b]) cudaFreeHost(pin[b]);
                cudaEventDestroy(ev[b]);
            }
        }
    } cleanup{pin, ev};
    std::fseek(fl.f, long(8 + 8 * row0 * n), SEEK_SET);
    int b = 0;
    for (int64_t r0 = 0; r0 < rows; r0 += chunk, b ^= 1) {
        const int64_t nr = std::min(chunk, rows - r0);
        RLRA_CUDA(cudaEventSynchronize(ev[b]));  // the previous copy out of this pinned buffer is done
        const size_t want = size_t(nr) * n;
        if (std::fread(pin[b], sizeof(double), want, fl.f) != want)
            raise(RLRA_EIO, fmt("load_binary: read from '%s' failed at byte offset %lld", path.c_str(),
                                8LL + 8LL * (row0 + r0) * n));
        RLRA_CUDA(cudaMemcpyAsync(stage[b].p, pin[b], sizeof(double) * want, cudaMemcpyHostToDevice, ctx.stream));
        RLRA_CUDA(cudaEventRecord(ev[b], ctx.stream));
        rowmajor_to_colmajor_kernel<<<grid_for(ctx, nr * n), 256, 0, ctx.stream>>>(
            stage[b].d(), int(nr), n, dst.p + r0, dst.ld, row0 + r0, static_cast<unsigned long long*>(bad.p));
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
    }
    unsigned long long first = 0;
    RLRA_CUDA(cudaMemcpyAsync(&first, bad.p, sizeof(first), cudaMemcpyDeviceToHost, ctx.stream));
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    if (first != ~0ull) {
        const long long i = (long long)(first / unsigned(n)), j = (long long)(first % unsigned(n));
        raise(RLRA_EIO, fmt("load_binary: '%s' holds a non-finite value at byte offset %lld (row %lld, column %lld)",
                            path.c_str(), 8LL + 8LL * (long long)first, i, j));
    }
}

void save_binary(Context& ctx, const std::string& path, const DMat& src) {
    const int m = int(src.rows), n = int(src.cols);
    File fl(path, "wb");
    if (!fl.f) raise(RLRA_EIO, fmt("save_binary: cannot open '%s' for writing", path.c_str()));
    unsigned char hdr[8];
    put_i32_le(hdr, m);
    put_i32_le(hdr + 4, n);
    if (std::fwrite(hdr, 1, 8, fl.f) != 8) raise(RLRA_EIO, fmt("save_binary: write to '%s' failed", path.c_str()));
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(std::max(m, 1), (int64_t(64) << 20) / (8LL * std::max(n, 1))));
    Buf stage(ctx, sizeof(double) * size_t(chunk) * std::max(n, 1));
    std::vector<double> host(size_t(chunk) * std::max(n, 1));
    for (int64_t r0 = 0; r0 < m; r0 += chunk) {
        const int64_t nr = std::min<int64_t>(chunk, m - r0);
        colmajor_to_rowmajor_kernel<<<grid_for(ctx, nr * n), 256, 0, ctx.stream>>>(src.p + r0, src.ld, int(nr), n,
                                                                                     stage.d());
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
        RLRA_CUDA(cudaMemcpyAsync(host.data(), stage.p, sizeof(double) * nr * n, cudaMemcpyDeviceToHost, ctx.stream));
        RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
        if (std::fwrite(host.data(), sizeof(double), size_t(nr) * n, fl.f) != size_t(nr) * n)
            raise(RLRA_EIO, fmt("save_binary: write to '%s' failed", path.c_str()));
    }
    if (std::fflush(fl.f) != 0) raise(RLRA_EIO, fmt("save_binary: write to '%s' failed", path.c_str()));
}

void gen_test_matrix(Context& ctx, const std::vector<double>& sigma, uint64_t seed, double noise, const DMat& A) {
    const int m = int(A.rows), n = int(A.cols), r = int(sigma.size());
    if (r > std::min(m, n)) raise(RLRA_EDIM, fmt("gen_test_matrix: %d singular values for a %dx%d matrix", r, m, n));
    if (r == 0) {
        zero_mat(ctx, A);
    } else {
        DMatBuf U(ctx, m, r), V(ctx, n, r);
        Buf s(ctx, sizeof(double) * r);
        philox_fill(ctx, U.m, seed, 101, 0);
        philox_fill(ctx, V.m, seed, 102, 0);
        orth_inplace(ctx, U.m, nullptr);
        orth_inplace(ctx, V.m, nullptr);
        RLRA_CUDA(cudaMemcpyAsync(s.p, sigma.data(), sizeof(double) * r, cudaMemcpyHostToDevice, ctx.stream));
        scale_cols_by_kernel<<<grid_for(ctx, int64_t(m) * r), 256, 0, ctx.stream>>>(U.m.p, U.m.ld, m, r, s.d());
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
        gemm(ctx, Op::N, Op::T, 1.0, U.m, V.m, 0.0, A);  // A = U diag(s) V^T
        RLRA_CUDA(cudaStreamSynchronize(ctx.stream));    // sigma (host) outlives its copy
    }
    if (noise != 0.0) {
        DMatBuf G(ctx, m, n);
        philox_fill(ctx, G.m, seed, 103, 0);
        axpy_mat_kernel<<<grid_for(ctx, int64_t(m) * n), 256, 0, ctx.stream>>>(A.p, A.ld, G.m.p, G.m.ld, m, n, noise);
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
    }
}

void gen_test_matrix_rowsharded(Context& ctx, Comm& cm, const std::vector<double>& sigma, uint64_t seed,
                                double noise, int64_t row0, int64_t m_total, const DMat& A) {
    const int mg = int(A.rows), n = int(A.cols), r = int(sigma.size());
    if (r > std::min<int64_t>(m_total, n))
        raise(RLRA_EDIM, fmt("gen_test_matrix: %d singular values for a %lldx%d matrix", r, (long long)m_total, n));
    if (r == 0) {
        zero_mat(ctx, A);
    } else {
        DMatBuf U(ctx, std::max(mg, 1), r), V(ctx, n, r);
        const DMat Ug = U.m.block(0, 0, mg, r);
        Buf s(ctx, sizeof(double) * r);
        if (mg > 0) philox_fill(ctx, Ug, seed, 101, row0);
        philox_fill(ctx, V.m, seed, 102, 0);
        orth_rowsharded(ctx, cm, Ug, m_total, false);
        orth_inplace(ctx, V.m, nullptr);
        if (mg > 0) {
            RLRA_CUDA(cudaMemcpyAsync(s.p, sigma.data(), sizeof(double) * r, cudaMemcpyHostToDevice, ctx.stream));
            scale_cols_by_kernel<<<grid_for(ctx, int64_t(mg) * r), 256, 0, ctx.stream>>>(Ug.p, Ug.ld, mg, r, s.d());
            RLRA_LAUNCH_CHECK();
            ++ctx.launches;
            gemm(ctx, Op::N, Op::T, 1.0, Ug, V.m, 0.0, A);
        }
        comm_sync(ctx, cm);  // sigma (host) outlives its copy
    }
    if (noise != 0.0 && mg > 0) {
        DMatBuf G(ctx, mg, n);
        philox_fill(ctx, G.m, seed, 103, row0);
        axpy_mat_kernel<<<grid_for(ctx, int64_t(mg) * n), 256, 0, ctx.stream>>>(A.p, A.ld, G.m.p, G.m.ld, mg, n, noise);
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
    }
}

VerifyReport verify_lowrank(Context& ctx, const DMat& A, const DMat& X, const DMat& Y, int k,
                            const std::vector<double>& sigma_true) {
    const int m = int(A.rows), n = int(A.cols);
    VerifyReport r;
    Buf sq(ctx, sizeof(double) * 2);
    sum_squares(ctx, A, sq.d());
    if (k > 0) {  // ||A - X Y^T||^2 through the fused residual GEMM
        GemmOpts o;
        o.epi = EPI_RESID;
        o.R = A.p;
        o.ldr = A.ld;
        o.resid_sq = sq.d() + 1;
        gemm(ctx, Op::N, Op::T, m, n, k, 1.0, X.p, X.ld, Y.p, Y.ld, 0.0, nullptr, 0, o);
    } else {
        sum_squares(ctx, A, sq.d() + 1);
    }
    RLRA_CUDA(cudaMemcpyAsync(ctx.h_scalars, sq.p, sizeof(double) * 2, cudaMemcpyDeviceToHost, ctx.stream));
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    const double fro_a = std::sqrt(ctx.h_scalars[0]);
    const double fro_diff = std::sqrt(ctx.h_scalars[1]);
    r.rel_frobenius_error = fro_diff / (fro_a > 0.0 ? fro_a : 1.0);
    if (fro_diff == 0.0) {
        r.rel_spectral_error = 0.0;
    } else {
        rlra_rng est;
        rlra_rng_seed(&est, 0x5bd1e995u);  // report.hpp:116: fixed, reproducible
        const DMat Xk = X.block(0, 0, m, k), Yk = Y.block(0, 0, n, k);
        const double spec_a = spectral_est(ctx, A, nullptr, nullptr, 60, &est);
        const double spec_d = spectral_est(ctx, A, k > 0 ? &Xk : nullptr, k > 0 ? &Yk : nullptr, 60, &est);
        r.rel_spectral_error = spec_d / (spec_a > 0.0 ? spec_a : 1.0);
    }
    if (!sigma_true.empty()) {  // report.hpp:123-136
        const int rr = int(sigma_true.size());
        double tail2 = 0.0, all2 = 0.0;
        for (int j = 0; j < rr; ++j) {
            all2 += sigma_true[j] * sigma_true[j];
            if (j >= k) tail2 += sigma_true[j] * sigma_true[j];
        }
        const double sig1 = sigma_true[0] > 0.0 ? sigma_true[0] : 1.0;
        const double sig_next = k < rr ? sigma_true[size_t(k)] : 0.0;
        r.fro_floor = all2 > 0.0 ? std::sqrt(tail2 / all2) : 0.0;
        r.spec_floor = sig_next / sig1;
        r.spec_bound = std::sqrt(double(k) * n) * sig_next / sig1;
    }
    return r;
}

VerifyReport verify_svd(Context& ctx, const DMat& A, const DMat& U, const double* sigma, const DMat& V, int k,
                        const std::vector<double>& sigma_true) {
    const int m = int(A.rows);
    DMatBuf US(ctx, m, std::max(k, 1));
    if (k > 0) {
        copy_mat(ctx, U.block(0, 0, m, k), US.m.block(0, 0, m, k));
        scale_cols_by_kernel<<<grid_for(ctx, int64_t(m) * k), 256, 0, ctx.stream>>>(US.m.p, US.m.ld, m, k, sigma);
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
    }
    return verify_lowrank(ctx, A, US.m, V, k, sigma_true);
}

// qb_single (qb.hpp:43-95): one Gaussian direction per step, projected
// against the captured basis, normalised, B row = y^T R, R -= y b^T; GEMV
// and rank-1 kernels over the residual copy (a BLAS-2 method by design)
__global__ void rank1_sub_kernel(double* R, int64_t ldr, int m, int n, const double* y, const double* b) {
    const int64_t tot = int64_t(m) * n;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e % m), j = int(e / m);
        R[i + int64_t(j) * ldr] -= y[i] * b[j];
    }
}

QbOut qb_single(Context& ctx, const DMat& A, double tol, int max_rank, OmegaSource& om, const DMat& Q, const DMat& B) {
    const int m = int(A.rows), n = int(A.cols);
    DMatBuf R(ctx, m, n);
    copy_mat(ctx, A, R.m);
    Buf om_d(ctx, sizeof(double) * n), t(ctx, sizeof(double) * std::max(max_rank, 1)), tmp(ctx, sizeof(double) * m),
        sc(ctx, sizeof(double) * 2);
    std::vector<double> h(n);
    QbOut out;
    out.reached = false;  // set when the residual drops below tol (qb.hpp:58-61)
    double resid = 0.0;
    {
        Buf s2(ctx, sizeof(double));
        sum_squares(ctx, R.m, s2.d());
        RLRA_CUDA(cudaMemcpyAsync(ctx.h_scalars, s2.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
        RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
        resid = std::sqrt(ctx.h_scalars[0]);
    }
    for (;;) {
        if (resid < tol) {
            out.reached = true;
            break;
        }
        if (out.ell >= max_rank) break;
        const int l = out.ell;
        double* y = Q.p + int64_t(l) * Q.ld;
        double ynorm = 0.0;
        for (int tries = 0;; ++tries) {
            const int draw = om.next_draw++;
            if (om.o->mode == RLRA_OMEGA_PHILOX) {
                DMat od{om_d.d(), n, 1, std::max(n, 1)};
                philox_fill(ctx, od, om.o->seed, draw, 0);
            } else {
                if (!om.o->fill) raise(RLRA_EINVAL, "rlra_omega: callback mode without a fill function");
                om.o->fill(om.o->user, draw, n, 1, h.data());
                RLRA_CUDA(cudaMemcpyAsync(om_d.p, h.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx.stream));
            }
            gemv(ctx, false, R.m, om_d.d(), y);  // y = R omega
            if (l > 0) {                          // y -= Q (Q^T y)
                const DMat Ql = Q.block(0, 0, m, l);
                gemv(ctx, true, Ql, y, t.d());
                gemv(ctx, false, Ql, t.d(), tmp.d());
                axpy_mat_kernel<<<grid_for(ctx, m), 256, 0, ctx.stream>>>(y, m, tmp.d(), m, m, 1, -1.0);
                RLRA_LAUNCH_CHECK();
            }
            ynorm = std::sqrt(sq_norm(ctx, y, m, sc.d()));
            if (ynorm >= 1e-14 * resid) break;
            if (tries + 1 >= 64)
                raise(RLRA_ENUM, fmt("qb_single: no new direction found in 64 draws (residual %g)", resid));
        }
        scale_vec_kernel<<<grid_for(ctx, m), 256, 0, ctx.stream>>>(y, m, sc.d());  // sc holds ||y||^2
        RLRA_LAUNCH_CHECK();
        // b = y^T R -> row l of B (stride B.ld), then R -= y b^T
        Buf bj(ctx, sizeof(double) * n);
        gemv(ctx, true, R.m, y, bj.d());
        RLRA_CUDA(cudaMemcpy2DAsync(B.p + l, sizeof(double) * B.ld, bj.p, sizeof(double), sizeof(double), n,
                                    cudaMemcpyDeviceToDevice, ctx.stream));
        rank1_sub_kernel<<<grid_for(ctx, int64_t(m) * n), 256, 0, ctx.stream>>>(R.m.p, R.m.ld, m, n, y, bj.d());
        RLRA_LAUNCH_CHECK();
        ctx.launches += 3;
        ++out.ell;
        Buf s2(ctx, sizeof(double));
        sum_squares(ctx, R.m, s2.d());
        RLRA_CUDA(cudaMemcpyAsync(ctx.h_scalars, s2.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
        RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
        resid = std::sqrt(ctx.h_scalars[0]);
        out.hist.push_back(resid);
    }
    out.final_residual = resid;
    return out;
}

}  // namespace rlra_b200
