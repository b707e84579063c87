// reduce.cu — deterministic reductions and small data-movement kernels.
#include "reduce.cuh"
#include "hostio.cuh"

namespace rlra_b200 {

namespace {

constexpr int kRedThreads = 512;

__device__ __forceinline__ double block_sum_fixed(double v, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        for (int i = 0; i < nw; ++i) t += sh[i];
    }
    return t;
}

__global__ void sum_kernel(const double* x, int64_t n, double* out) {
    __shared__ double sh[32];
    double v = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v += x[i];
    const double t = block_sum_fixed(v, sh);
    if (threadIdx.x == 0) *out = t;
}

// per-block partial of sum A(i,j)^2 with a fixed element->thread mapping
__global__ void sumsq_partial_kernel(const double* a, int64_t m, int64_t n, int64_t ld,
                                     double* partial) {
    __shared__ double sh[32];
    const int64_t total = m * n;
    double v = 0.0;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const double x = a[(e % m) + (e / m) * ld];
        v += x * x;
    }
    const double t = block_sum_fixed(v, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

template <class F>
__global__ void map2d_kernel(int64_t m, int64_t n, F f) {
    const int64_t total = m * n;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x)
        f(e % m, e / m);
}

template <class F>
void map2d(Context& ctx, int64_t m, int64_t n, F f) {
    if (m <= 0 || n <= 0) return;
    const int64_t total = m * n;
    const int blocks = int(std::min<int64_t>((total + 255) / 256, int64_t(ctx.num_sms) * 16));
    map2d_kernel<<<blocks, 256, 0, ctx.stream>>>(m, n, f);
    RLRA_LAUNCH_CHECK();
    ++ctx.launches;
}

}  // namespace

void sum_fixed_order(Context& ctx, const double* x, int64_t n, double* out) {
    sum_kernel<<<1, kRedThreads, 0, ctx.stream>>>(x, n, out);
    RLRA_LAUNCH_CHECK();
    ++ctx.launches;
}

void sum_squares(Context& ctx, const DMat& a, double* out_sq) {
    const int64_t total = a.rows * a.cols;
    if (total == 0) {
        RLRA_CUDA(cudaMemsetAsync(out_sq, 0, sizeof(double), ctx.stream));
        return;
    }
    const int blocks = int(std::min<int64_t>((total + 255) / 256, int64_t(ctx.num_sms) * 4));
    Buf part(ctx, sizeof(double) * blocks);
    sumsq_partial_kernel<<<blocks, 256, 0, ctx.stream>>>(a.p, a.rows, a.cols, a.ld, part.d());
    RLRA_LAUNCH_CHECK();
    ++ctx.launches;
    sum_fixed_order(ctx, part.d(), blocks, out_sq);
}

void copy_mat(Context& ctx, const DMat& s, const DMat& d) {
    const double* sp = s.p;
    double* dp = d.p;
    const int64_t sl = s.ld, dl = d.ld;
    map2d(ctx, s.rows, s.cols,
          [=] __device__(int64_t i, int64_t j) { dp[i + j * dl] = sp[i + j * sl]; });
}

void transpose_mat(Context& ctx, const DMat& s, const DMat& d) {
    const double* sp = s.p;
    double* dp = d.p;
    const int64_t sl = s.ld, dl = d.ld;
    // iterate over destination so writes are coalesced
    map2d(ctx, d.rows, d.cols,
          [=] __device__(int64_t i, int64_t j) { dp[i + j * dl] = sp[j + i * sl]; });
}

void zero_mat(Context& ctx, const DMat& d) {
    double* dp = d.p;
    const int64_t dl = d.ld;
    map2d(ctx, d.rows, d.cols, [=] __device__(int64_t i, int64_t j) { dp[i + j * dl] = 0.0; });
}

void eye_mat(Context& ctx, const DMat& d) {
    double* dp = d.p;
    const int64_t dl = d.ld;
    map2d(ctx, d.rows, d.cols,
          [=] __device__(int64_t i, int64_t j) { dp[i + j * dl] = i == j ? 1.0 : 0.0; });
}

void gather_cols(Context& ctx, const DMat& s, const int* idx, int count, const DMat& d) {
    const double* sp = s.p;
    double* dp = d.p;
    const int64_t sl = s.ld, dl = d.ld;
    map2d(ctx, s.rows, count,
          [=] __device__(int64_t i, int64_t j) { dp[i + j * dl] = sp[i + int64_t(idx[j]) * sl]; });
}

void gather_rows(Context& ctx, const DMat& s, const int* idx, int count, const DMat& d) {
    const double* sp = s.p;
    double* dp = d.p;
    const int64_t sl = s.ld, dl = d.ld;
    map2d(ctx, count, s.cols,
          [=] __device__(int64_t i, int64_t j) { dp[i + j * dl] = sp[int64_t(idx[i]) + j * sl]; });
}

void sub_inplace(Context& ctx, const DMat& y, const DMat& x) {
    double* yp = y.p;
    const double* xp = x.p;
    const int64_t yl = y.ld, xl = x.ld;
    map2d(ctx, y.rows, y.cols,
          [=] __device__(int64_t i, int64_t j) { yp[i + j * yl] = yp[i + j * yl] - xp[i + j * xl]; });
}

void symmetrize_upper(Context& ctx, const DMat& a) {
    double* p = a.p;
    const int64_t l = a.ld;
    map2d(ctx, a.rows, a.cols, [=] __device__(int64_t i, int64_t j) {
        if (i > j) p[i + j * l] = p[j + i * l];
    });
}

void h2d_mat(Context& ctx, const double* h, int64_t ldh, const DMat& d) {
    h2d_copy(ctx, ctx.stream, h, ldh, d);  // pageable host memory is staged (hostio.cu)
}

void d2h_mat(Context& ctx, const DMat& d, double* h, int64_t ldh) {
    d2h_copy(ctx, d, h, ldh);  // returns with h filled
}

}  // namespace rlra_b200
