// cpqr.cu — column-pivoted QR on the sketch (K8) and the clamped triangular
// solve (K9).
#include <cooperative_groups.h>

#include <cfloat>
#include <climits>

#include "cpqr.cuh"
#include "gemm.cuh"
#include "qr.cuh"
#include "reduce.cuh"

namespace cg = cooperative_groups;

namespace rlra_b200 {

namespace {

constexpr int kCpqrThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// (value desc, position asc) — the reference's strict '>' scan from f
// (core/qr.hpp:179-181) selects the largest value and, among equal values,
// the earliest position.
__device__ __forceinline__ bool better(double v, int p, double bv, int bp) {
    return v > bv || (v == bv && p < bp);
}

struct CpqrArgs {
    unsigned* bar;  // grid_sync state (Context::gbar)
    double* W;
    int64_t ldw;
    int m, n, kmax, rmax;
    int tol_mode;
    double tol;
    double* Vst;  // m x kmax, ld m
    double* beta;
    int* perm;
    double* cn;
    double* rn;
    double* slot_v;
    int* slot_p;
    double* slot_t;
    int* out;  // [0] frank, [1] reached, [2] degenerate
    double* res;
};

__global__ void __launch_bounds__(kCpqrThreads) cpqr_coop_kernel(CpqrArgs a) {
    __shared__ double sv[32], st[32];
    __shared__ int sp[32];
    __shared__ double shb[32];
    __shared__ int s_piv;
    const int G = gridDim.x, g = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int m = a.m, n = a.n;
    double* W = a.W;
    const int64_t ldw = a.ldw;
    const int cpb = (n + G - 1) / G;
    const int j0 = g * cpb, j1 = min(n, j0 + cpb);

    // block-level merge of per-warp (best, trailing) into the CTA slot
    auto publish = [&](double bv, int bp, double tr) {
        if (lane == 0) {
            sv[warp] = bv;
            sp[warp] = bp;
            st[warp] = tr;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double v = -DBL_MAX, t = 0.0;
            int p = INT_MAX;
            for (int w = 0; w < nw; ++w) {
                if (better(sv[w], sp[w], v, p)) {
                    v = sv[w];
                    p = sp[w];
                }
                t += st[w];
            }
            a.slot_v[g] = v;
            a.slot_p[g] = p;
            a.slot_t[g] = t;
        }
        __syncthreads();
    };

    // init: perm, squared norms (core/qr.hpp:157-161)
    {
        double bv = -DBL_MAX, tr = 0.0;
        int bp = INT_MAX;
        for (int j = j0 + warp; j < j1; j += nw) {
            double s = 0.0;
            for (int i = lane; i < m; i += 32) {
                const double x = W[i + int64_t(j) * ldw];
                s += x * x;
            }
            s = warp_sum(s);
            if (lane == 0) {
                a.perm[j] = j;
                a.cn[j] = s;
                a.rn[j] = s;
            }
            if (better(s, j, bv, bp)) {
                bv = s;
                bp = j;
            }
            tr += s;
        }
        publish(bv, bp, tr);
    }
    grid_sync(a.bar);

    int frank = 0;
    bool reached = false;
    if (a.tol_mode) {
        double t = 0.0;
        for (int c = 0; c < G; ++c) t += a.slot_t[c];
        const double r = sqrt(t);
        reached = r <= a.tol;
        if (g == 0 && threadIdx.x == 0) *a.res = r;
    }
    while (!reached && frank < a.kmax) {
        const int f = frank;
        if (g == 0) {
            if (threadIdx.x == 0) {
                double v = -DBL_MAX;
                int p = INT_MAX;
                for (int c = 0; c < G; ++c)
                    if (better(a.slot_v[c], a.slot_p[c], v, p)) {
                        v = a.slot_v[c];
                        p = a.slot_p[c];
                    }
                s_piv = p;
            }
            __syncthreads();
            const int piv = s_piv;
            if (piv != f) {  // core/qr.hpp:182-187
                for (int i = threadIdx.x; i < m; i += blockDim.x) {
                    const double t = W[i + int64_t(f) * ldw];
                    W[i + int64_t(f) * ldw] = W[i + int64_t(piv) * ldw];
                    W[i + int64_t(piv) * ldw] = t;
                }
                if (threadIdx.x == 0) {
                    int ti = a.perm[f];
                    a.perm[f] = a.perm[piv];
                    a.perm[piv] = ti;
                    double td = a.cn[f];
                    a.cn[f] = a.cn[piv];
                    a.cn[piv] = td;
                    td = a.rn[f];
                    a.rn[f] = a.rn[piv];
                    a.rn[piv] = td;
                }
                __syncthreads();
            }
            // householder_step on column f (core/qr.hpp:44-66)
            double s = 0.0;
            for (int i = f + threadIdx.x; i < m; i += blockDim.x) {
                const double x = W[i + int64_t(f) * ldw];
                s += x * x;
            }
            s = warp_sum(s);
            if (lane == 0) shb[warp] = s;
            __syncthreads();
            double norm2 = 0.0;
            for (int w = 0; w < nw; ++w) norm2 += shb[w];
            const double x1 = W[f + int64_t(f) * ldw];
            const double norm = sqrt(norm2);
            const bool zero = norm < 1e-300;
            const double alpha = x1 >= 0.0 ? -norm : norm;
            const double beta = zero ? 0.0 : 2.0 / (2.0 * (norm2 - alpha * x1));
            __syncthreads();
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                double vi = 0.0;
                if (!zero) vi = i > f ? W[i + int64_t(f) * ldw] : (i == f ? x1 - alpha : 0.0);
                a.Vst[i + int64_t(f) * m] = vi;
            }
            __syncthreads();
            for (int i = f + threadIdx.x; i < m; i += blockDim.x)
                W[i + int64_t(f) * ldw] = (i == f) ? (zero ? 0.0 : alpha) : 0.0;
            if (threadIdx.x == 0) {
                a.beta[f] = beta;
                if (zero) a.out[2] = 1;
            }
        }
        grid_sync(a.bar);
        // apply H_f to own trailing positions, downdate (core/qr.hpp:190-200)
        const double beta = a.beta[f];
        const double* v = a.Vst + int64_t(f) * m;
        double bv = -DBL_MAX, tr = 0.0;
        int bp = INT_MAX;
        for (int j = max(j0, f + 1) + warp; j < j1; j += nw) {
            double* wj = W + int64_t(j) * ldw;
            if (beta != 0.0) {
                double s = 0.0;
                for (int i = f + lane; i < m; i += 32) s += v[i] * wj[i];
                const double fct = beta * warp_sum(s);
                for (int i = f + lane; i < m; i += 32) wj[i] -= fct * v[i];
                __syncwarp();
            }
            const double d = wj[f];
            double c = a.cn[j] - d * d;
            const double ref = a.rn[j];
            double rr = ref;
            if (c < 1e-6 * ref || a.tol_mode) {
                double s = 0.0;
                for (int i = f + 1 + lane; i < m; i += 32) s += wj[i] * wj[i];
                s = warp_sum(s);
                if (c < 1e-6 * ref) {
                    c = s;
                    rr = s;
                }
                tr += s;
            }
            if (lane == 0) {
                a.cn[j] = c;
                a.rn[j] = rr;
            }
            if (better(c, j, bv, bp)) {
                bv = c;
                bp = j;
            }
        }
        publish(bv, bp, tr);
        ++frank;
        grid_sync(a.bar);
        if (a.tol_mode && frank < a.rmax) {
            double t = 0.0;
            for (int c = 0; c < G; ++c) t += a.slot_t[c];
            const double r = sqrt(t);
            if (g == 0 && threadIdx.x == 0) *a.res = r;
            if (r <= a.tol) reached = true;
        }
    }
    if (g == 0 && threadIdx.x == 0) {
        a.out[0] = frank;
        a.out[1] = reached ? 1 : 0;
    }
}

// S1 = W(0:f, :) with diag sign fix; Q1 columns flipped alongside.
__global__ void cpqr_finish_kernel(const double* W, int64_t ldw, int f, int n, double* S1,
                                   int64_t lds) {
    const int64_t tot = int64_t(f) * n;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e % f), j = int(e / f);
        const double s = W[i + int64_t(i) * ldw] < 0.0 ? -1.0 : 1.0;
        S1[i + int64_t(j) * lds] = s * W[i + int64_t(j) * ldw];
    }
}

__global__ void flip_cols_kernel(const double* W, int64_t ldw, int f, int m, double* Q, int64_t ldq) {
    const int64_t tot = int64_t(m) * f;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e % m), j = int(e / m);
        if (W[j + int64_t(j) * ldw] < 0.0) Q[i + int64_t(j) * ldq] = -Q[i + int64_t(j) * ldq];
    }
}

// trailing ||W(f:m, f:n)||^2 partial per block (fixed order)
__global__ void trailing_sq_kernel(const double* W, int64_t ldw, int m, int n, int f, double* part) {
    __shared__ double sh[32];
    const int mm = m - f, nn = n - f;
    double v = 0.0;
    if (mm > 0 && nn > 0) {
        const int64_t tot = int64_t(mm) * nn;
        for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot;
             e += int64_t(gridDim.x) * blockDim.x) {
            const double x = W[(f + e % mm) + (f + e / mm) * ldw];
            v += x * x;
        }
    }
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += sh[w];
        part[blockIdx.x] = t;
    }
}

// ---------------------------------------------------------- tri-solve ---
// One warp per right-hand side: column-oriented back substitution in shared
// memory.  t_i = b_i / s_ii, then b[0:i] -= t_i * S(0:i, i) (coalesced column).
__global__ void trisolve_kernel(const double* S, int64_t lds, int k, const double* B, int64_t ldb,
                                int nc, double* T, int64_t ldt) {
    extern __shared__ double xs[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    double* x = xs + int64_t(warp) * k;
    for (int j = blockIdx.x * wpb + warp; j < nc; j += gridDim.x * wpb) {
        for (int i = lane; i < k; i += 32) x[i] = B[i + int64_t(j) * ldb];
        __syncwarp();
        for (int i = k - 1; i >= 0; --i) {
            const double ti = x[i] / S[i + int64_t(i) * lds];
            __syncwarp();
            if (lane == 0) x[i] = ti;
            const double* si = S + int64_t(i) * lds;
            for (int r = lane; r < i; r += 32) x[r] -= ti * si[r];
            __syncwarp();
        }
        for (int i = lane; i < k; i += 32) T[i + int64_t(j) * ldt] = x[i];
        __syncwarp();
    }
}

__global__ void clamp_kernel(double* T, int64_t ldt, int k, int nc) {
    const int64_t tot = int64_t(k) * nc;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot;
         e += int64_t(gridDim.x) * blockDim.x) {
        double* p = T + (e % k) + (e / k) * ldt;
        if (fabs(*p) > 1e4) *p = *p > 0.0 ? 1e4 : -1e4;
    }
}

__global__ void diag_abs_kernel(const double* S, int64_t lds, int k, double* d) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x)
        d[i] = fabs(S[i + int64_t(i) * lds]);
}

}  // namespace

CpqrResult pivoted_qr(Context& ctx, const DMat& A, int k, double tol, const DMat* Q1, const DMat& S1,
                      int* perm) {
    const int m = int(A.rows), n = int(A.cols);
    const int rmax = std::min(m, n);
    const bool tol_mode = (k == 0 && tol > 0.0);
    if (!tol_mode && (k < 1 || k > rmax || tol != 0.0))
        raise(RLRA_EDIM, fmt("pivoted_qr_partial: need either k in [1,%d] with tol=0 or k=0 with "
                             "tol>0 (got k=%d, tol=%g)",
                             rmax, k, tol));
    const int kmax = tol_mode ? rmax : k;
    ProfScope prof(ctx, "cpqr", m, n, kmax, 0.0);
    DMatBuf W(ctx, m, n);
    copy_mat(ctx, A, W);
    Buf Vst(ctx, sizeof(double) * size_t(m) * std::max(kmax, 1)), beta(ctx, sizeof(double) * (kmax + 1)),
        cn(ctx, sizeof(double) * n), rn(ctx, sizeof(double) * n), out(ctx, sizeof(int) * 4),
        res(ctx, sizeof(double));
    int per_sm = 0;
    RLRA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cpqr_coop_kernel, kCpqrThreads, 0));
    int G = std::max(1, std::min(ctx.num_sms * std::max(1, per_sm), ceil_div(n, 4 * (kCpqrThreads / 32))));
    G = std::min(G, ctx.num_sms);
    Buf sv(ctx, sizeof(double) * G), sp(ctx, sizeof(int) * G), stt(ctx, sizeof(double) * G);
    RLRA_CUDA(cudaMemsetAsync(out.p, 0, sizeof(int) * 4, ctx.stream));
    RLRA_CUDA(cudaMemsetAsync(res.p, 0, sizeof(double), ctx.stream));
    CpqrArgs a;
    a.W = W.m.p;
    a.ldw = W.m.ld;
    a.m = m;
    a.n = n;
    a.kmax = kmax;
    a.rmax = rmax;
    a.tol_mode = tol_mode;
    a.tol = tol;
    a.Vst = Vst.d();
    a.beta = beta.d();
    a.perm = perm;
    a.cn = cn.d();
    a.rn = rn.d();
    a.slot_v = sv.d();
    a.slot_p = sp.i();
    a.slot_t = stt.d();
    a.out = out.i();
    a.res = res.d();
    a.bar = ctx.gbar;
    void* args[] = {&a};
    RLRA_CUDA(cudaLaunchCooperativeKernel((void*)cpqr_coop_kernel, dim3(G), dim3(kCpqrThreads), args,
                                          0, ctx.stream));
    ++ctx.launches;
    int h_out[4];
    double h_res = 0.0;
    RLRA_CUDA(cudaMemcpyAsync(h_out, out.p, sizeof(int) * 4, cudaMemcpyDeviceToHost, ctx.stream));
    RLRA_CUDA(cudaMemcpyAsync(&h_res, res.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    CpqrResult r;
    r.frank = h_out[0];
    r.reached = h_out[1] != 0;
    r.degenerate = h_out[2] != 0;
    const int f = r.frank;
    if (f > 0) {
        const int blocks = int(std::min<int64_t>((int64_t(f) * n + 255) / 256, int64_t(ctx.num_sms) * 8));
        cpqr_finish_kernel<<<blocks, 256, 0, ctx.stream>>>(W.m.p, W.m.ld, f, n, S1.p, S1.ld);
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
    }
    const bool need_q = Q1 != nullptr || (tol_mode && !r.reached);
    DMatBuf Qtmp;
    DMat Q;
    if (need_q && f > 0) {
        if (Q1) {
            Q = Q1->block(0, 0, m, f);
        } else {
            Qtmp = DMatBuf(ctx, m, f);
            Q = Qtmp.m;
        }
        form_q(ctx, Vst.d(), m, beta.d(), m, f, Q);
        const int blocks = int(std::min<int64_t>((int64_t(m) * f + 255) / 256, int64_t(ctx.num_sms) * 8));
        flip_cols_kernel<<<blocks, 256, 0, ctx.stream>>>(W.m.p, W.m.ld, f, m, Q.p, Q.ld);
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
    }
    if (!tol_mode) {
        // exact trailing norm (core/qr.hpp:163-168,222-224)
        const int blocks = ctx.num_sms;
        Buf part(ctx, sizeof(double) * blocks), tot(ctx, sizeof(double));
        trailing_sq_kernel<<<blocks, 256, 0, ctx.stream>>>(W.m.p, W.m.ld, m, n, f, part.d());
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
        sum_fixed_order(ctx, part.d(), blocks, tot.d());
        RLRA_CUDA(cudaMemcpyAsync(&h_res, tot.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
        RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
        r.residual = sqrt(h_res);
        r.reached = false;
    } else if (r.reached) {
        r.residual = h_res;
    } else {
        // ||A(:,perm) - Q1 S1||_F at full rank (core/qr.hpp:229-233)
        DMatBuf Ap(ctx, m, n);
        gather_cols(ctx, A, perm, n, Ap);
        Buf sq(ctx, sizeof(double));
        GemmOpts o;
        o.epi = EPI_RESID;
        o.R = Ap.m.p;
        o.ldr = Ap.m.ld;
        o.resid_sq = sq.d();
        gemm(ctx, Op::N, Op::N, m, n, f, 1.0, Q.p, Q.ld, S1.p, S1.ld, 0.0, nullptr, 0, o);
        RLRA_CUDA(cudaMemcpyAsync(&h_res, sq.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
        RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
        r.residual = sqrt(h_res);
        r.reached = r.residual <= tol;
    }
    return r;
}

bool upper_tri_solve(Context& ctx, const DMat& S11, const DMat& S12, const DMat& T) {
    const int k = int(S11.rows), nc = int(S12.cols);
    if (S11.cols != k)
        raise(RLRA_EDIM, fmt("upper_tri_solve: S11 is %dx%d, need square", k, int(S11.cols)));
    if (S12.rows != k)
        raise(RLRA_EDIM, fmt("upper_tri_solve: S12 has %d rows, need %d", int(S12.rows), k));
    if (k == 0) return false;
    Buf d(ctx, sizeof(double) * k);
    diag_abs_kernel<<<ceil_div(k, 256), 256, 0, ctx.stream>>>(S11.p, S11.ld, k, d.d());
    RLRA_LAUNCH_CHECK();
    ++ctx.launches;
    std::vector<double> hd(k);
    RLRA_CUDA(cudaMemcpyAsync(hd.data(), d.p, sizeof(double) * k, cudaMemcpyDeviceToHost, ctx.stream));
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    double dmax = 0.0, dmin = INFINITY;
    for (int i = 0; i < k; ++i) {
        if (hd[i] == 0.0)
            raise(RLRA_ENUM, fmt("upper_tri_solve: zero diagonal at position %d", i));
        dmax = std::max(dmax, hd[i]);
        dmin = std::min(dmin, hd[i]);
    }
    if (nc > 0) {
        int wpb = int(std::max<int64_t>(1, std::min<int64_t>(8, (160 * 1024) / (int64_t(k) * 8))));
        const size_t smem = sizeof(double) * size_t(k) * wpb;
        if (smem > 227 * 1024) raise(RLRA_EDIM, fmt("upper_tri_solve: k=%d too large", k));
        RLRA_CUDA(cudaFuncSetAttribute(trisolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(smem)));
        const int blocks = std::max(1, std::min(ctx.num_sms * 2, ceil_div(nc, wpb)));
        trisolve_kernel<<<blocks, wpb * 32, smem, ctx.stream>>>(S11.p, S11.ld, k, S12.p, S12.ld, nc,
                                                                T.p, T.ld);
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
    }
    if (dmax / dmin > 1e12) {
        if (nc > 0) {
            const int blocks = int(std::min<int64_t>((int64_t(k) * nc + 255) / 256, int64_t(ctx.num_sms) * 8));
            clamp_kernel<<<blocks, 256, 0, ctx.stream>>>(T.p, T.ld, k, nc);
            RLRA_LAUNCH_CHECK();
            ++ctx.launches;
        }
        return true;
    }
    return false;
}

}  // namespace rlra_b200
