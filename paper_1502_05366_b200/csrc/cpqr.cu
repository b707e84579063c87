// cpqr.cu — column-pivoted QR on the sketch (K8) and the clamped triangular
// solve (K9).
#include <cooperative_groups.h>

#include <cfloat>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "cpqr.cuh"
#include "gemm.cuh"
#include "qr.cuh"
#include "reduce.cuh"

namespace cg = cooperative_groups;

namespace rlra_b200 {

namespace {

constexpr int kCpqrThreads = 256;
constexpr int kCpqrStepThreads = 384;  // 12 warps: more L2 round trips in flight per SM
constexpr int kCpqrRegs = 24;  // register-resident rows per lane in cpqr_step_kernel (m - f <= 768)

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
    long long* phase_clk;  // optional: CTA 0's clock64 per step phase (RLRA_CPQR_PHASES)
    // cpqr_res_kernel only
    int* slot_s;       // 2 x G candidate storage columns
    double* slot_col;  // 2 x G x m candidate column data
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

// ------------------------------------------------ one barrier per pivot ---
// The same Businger–Golub steps as cpqr_coop_kernel (identical arithmetic,
// so identical pivots), reorganised so a step needs ONE grid barrier and no
// single-CTA phase: columns stay where they are (storage s = original column
// index; the norms travel with them) and every CTA keeps the position <->
// storage maps in shared memory and applies each swap itself.  Per step every
// CTA (1) reduces the G slots to the pivot, (2) reads the pivot column (rows
// f..m) and forms H_f in shared memory — the same reduction order in every
// CTA, so every CTA holds the same v, beta — and (3) applies H_f to its own
// trailing storage columns and downdates their norms (core/qr.hpp:190-200).
// The pivot column's own rows f..m become (alpha, 0, ...) at the start of the
// next step (nobody reads them before).  W is left in storage order; the host
// gathers it into position order afterwards.
__global__ void __launch_bounds__(kCpqrStepThreads) cpqr_step_kernel(CpqrArgs a) {
    extern __shared__ double csm[];
    const int m = a.m, n = a.n;
    const int G = gridDim.x, g = blockIdx.x, t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31, nw = blockDim.x >> 5;
    double* W = a.W;
    const int64_t ldw = a.ldw;
    const int cpb = (n + G - 1) / G;
    const int j0 = g * cpb, j1 = min(n, j0 + cpb);
    double* vsh = csm;                                         // m: H_f's vector
    double* cnS = csm + m;                                     // own columns' norms (owner-only state)
    double* rnS = cnS + cpb;
    int* p2s = reinterpret_cast<int*>(rnS + cpb);              // position -> storage
    int* s2p = p2s + n;                                        // storage -> position
    __shared__ double sv[32], st[32], shb[32];
    __shared__ int sp[32];
    __shared__ int s_piv;
    for (int i = t; i < n; i += blockDim.x) p2s[i] = s2p[i] = i;
    const bool clk = a.phase_clk != nullptr && g == 0 && t == 0;
    long long ph[5] = {0, 0, 0, 0, 0}, c0 = clock64();
    auto mark = [&](int i) {
        if (clk) {
            const long long c1 = clock64();
            ph[i] += c1 - c0;
            c0 = c1;
        }
    };

    // slots are double-buffered by step parity: step f reads buffer f & 1
    // (published during step f - 1) while fast CTAs already publish step f's
    // candidates into the other buffer — with one barrier per step a single
    // buffer would let a fast CTA overwrite a slot a slow CTA has not read yet
    int par = 0;
    auto publish = [&](double bv, int bp, double tr) {
        if (lane == 0) {
            sv[warp] = bv;
            sp[warp] = bp;
            st[warp] = tr;
        }
        __syncthreads();
        if (t == 0) {
            double v = -DBL_MAX, tt = 0.0;
            int p = INT_MAX;
            for (int w = 0; w < nw; ++w) {
                if (better(sv[w], sp[w], v, p)) {
                    v = sv[w];
                    p = sp[w];
                }
                tt += st[w];
            }
            a.slot_v[par * G + g] = v;
            a.slot_p[par * G + g] = p;
            a.slot_t[par * G + g] = tt;
        }
        __syncthreads();
    };

    {  // squared norms (core/qr.hpp:157-161)
        double bv = -DBL_MAX, tr = 0.0;
        int bp = INT_MAX;
        for (int j = j0 + warp; j < j1; j += nw) {
            double sum = 0.0;
            for (int i = lane; i < m; i += 32) {
                const double x = W[i + int64_t(j) * ldw];
                sum += x * x;
            }
            sum = warp_sum(sum);
            if (lane == 0) {
                cnS[j - j0] = sum;
                rnS[j - j0] = sum;
            }
            if (better(sum, j, bv, bp)) {
                bv = sum;
                bp = j;
            }
            tr += sum;
        }
        publish(bv, bp, tr);
    }
    grid_sync(a.bar);

    int frank = 0;
    bool reached = false;
    if (a.tol_mode) {
        double tt = 0.0;
        for (int c = 0; c < G; ++c) tt += a.slot_t[c];
        const double r = sqrt(tt);
        reached = r <= a.tol;
        if (g == 0 && t == 0) *a.res = r;
    }
    int pend_s = -1, pend_f = 0;  // the pivot column whose rows pend_f.. become (alpha, 0, ...)
    double pend_alpha = 0.0;
    auto finish_pending = [&]() {
        if (pend_s >= 0) {
            double* col = W + int64_t(pend_s) * ldw;
            for (int i = pend_f + t; i < m; i += blockDim.x) col[i] = (i == pend_f) ? pend_alpha : 0.0;
            pend_s = -1;
        }
    };
    while (!reached && frank < a.kmax) {
        const int f = frank;
        finish_pending();
        // 1. pivot (value desc, position asc) over the CTA slots
        if (warp == 0) {
            double v = -DBL_MAX;
            int p = INT_MAX;
            for (int c = lane; c < G; c += 32)
                if (better(a.slot_v[par * G + c], a.slot_p[par * G + c], v, p)) {
                    v = a.slot_v[par * G + c];
                    p = a.slot_p[par * G + c];
                }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, v, o);
                const int op = __shfl_xor_sync(0xffffffffu, p, o);
                if (better(ov, op, v, p)) {
                    v = ov;
                    p = op;
                }
            }
            if (lane == 0) s_piv = p;
        }
        __syncthreads();
        const int piv = s_piv;
        const int sf = p2s[f], spv = p2s[piv];
        mark(0);
        // 2. householder_step on the pivot column (core/qr.hpp:44-66), in every CTA
        const double* pc = W + int64_t(spv) * ldw;
        double sum = 0.0;
        for (int i = f + t; i < m; i += blockDim.x) {
            const double x = pc[i];
            vsh[i] = x;
            sum += x * x;
        }
        sum = warp_sum(sum);
        if (lane == 0) shb[warp] = sum;
        __syncthreads();
        double norm2 = 0.0;
        for (int w = 0; w < nw; ++w) norm2 += shb[w];
        const double x1 = vsh[f];
        const double norm = sqrt(norm2);
        const bool zero = norm < 1e-300;
        const double alpha = x1 >= 0.0 ? -norm : norm;
        const double beta = zero ? 0.0 : 2.0 / (2.0 * (norm2 - alpha * x1));
        __syncthreads();
        if (zero) {
            for (int i = f + t; i < m; i += blockDim.x) vsh[i] = 0.0;
        } else if (t == 0) {
            vsh[f] = x1 - alpha;
        }
        // the swap (core/qr.hpp:182-187), on the maps
        if (t == 0 && piv != f) {
            p2s[f] = spv;
            p2s[piv] = sf;
            s2p[spv] = f;
            s2p[sf] = piv;
        }
        __syncthreads();
        if (g == 0) {
            for (int i = t; i < m; i += blockDim.x) a.Vst[i + int64_t(f) * m] = i < f ? 0.0 : vsh[i];
            if (t == 0) {
                a.beta[f] = beta;
                if (zero) a.out[2] = 1;
            }
        }
        mark(1);
        par ^= 1;  // this step's candidates go to the other buffer
        // 3. apply H_f to own trailing columns, downdate (core/qr.hpp:190-200).
        // Columns up to 32 * kCpqrRegs rows below f are held in registers, two
        // per warp at a time, so the L2 round trips overlap (the same
        // arithmetic in the same order as the loop form below).
        double bv = -DBL_MAX, tr = 0.0;
        int bp = INT_MAX;
        auto downdate = [&](int j, int pos, double d, double s2) {
            double c = cnS[j - j0] - d * d;
            const double ref = rnS[j - j0];
            double rr = ref;
            if (c < 1e-6 * ref || a.tol_mode) {
                if (c < 1e-6 * ref) {
                    c = s2;
                    rr = s2;
                }
                tr += s2;
            }
            __syncwarp();
            if (lane == 0) {
                cnS[j - j0] = c;
                rnS[j - j0] = rr;
            }
            __syncwarp();
            if (better(c, pos, bv, bp)) {
                bv = c;
                bp = pos;
            }
        };
        if (m - f <= 32 * kCpqrRegs) {
            // row chunks below f still live (warp-uniform): the rest are zero
            // on both sides and are skipped instead of loaded and multiplied
            const int UR = (m - f + 31) >> 5;
            for (int j = j0 + warp; j < j1; j += 2 * nw) {
                const int jj[2] = {j, j + nw};
                bool on[2];
                double x[2][kCpqrRegs];
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    on[b] = jj[b] < j1 && s2p[jj[b]] > f;
                    const double* wj = W + int64_t(on[b] ? jj[b] : 0) * ldw;
#pragma unroll
                    for (int u = 0; u < kCpqrRegs; ++u) {
                        const int i = f + lane + 32 * u;
                        x[b][u] = (u < UR && on[b] && i < m) ? wj[i] : 0.0;
                    }
                }
                if (beta != 0.0) {
                    double sd[2] = {0.0, 0.0};
#pragma unroll
                    for (int u = 0; u < kCpqrRegs; ++u) {
                        if (u >= UR) break;
                        const int i = f + lane + 32 * u;
                        const double vi = i < m ? vsh[i] : 0.0;
#pragma unroll
                        for (int b = 0; b < 2; ++b) sd[b] += vi * x[b][u];
                    }
#pragma unroll
                    for (int b = 0; b < 2; ++b) {
                        const double fct = beta * warp_sum(sd[b]);
#pragma unroll
                        for (int u = 0; u < kCpqrRegs; ++u) {
                            const int i = f + lane + 32 * u;
                            if (u < UR && i < m) x[b][u] -= fct * vsh[i];
                        }
                    }
#pragma unroll
                    for (int b = 0; b < 2; ++b) {
                        if (!on[b]) continue;
                        double* wj = W + int64_t(jj[b]) * ldw;
#pragma unroll
                        for (int u = 0; u < kCpqrRegs; ++u) {
                            const int i = f + lane + 32 * u;
                            if (u < UR && i < m) wj[i] = x[b][u];
                        }
                    }
                }
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    const double d = __shfl_sync(0xffffffffu, x[b][0], 0);  // row f
                    double s2 = 0.0;
                    const double c0 = cnS[on[b] ? jj[b] - j0 : 0] - d * d, r0 = rnS[on[b] ? jj[b] - j0 : 0];
                    if (c0 < 1e-6 * r0 || a.tol_mode) {  // uniform across the warp
#pragma unroll
                        for (int u = 0; u < kCpqrRegs; ++u) {
                            const int i = f + lane + 32 * u;
                            if (i > f && i < m) s2 += x[b][u] * x[b][u];
                        }
                        s2 = warp_sum(s2);
                    }
                    if (on[b]) downdate(jj[b], s2p[jj[b]], d, s2);
                }
            }
        } else {
            for (int j = j0 + warp; j < j1; j += nw) {
                const int pos = s2p[j];
                if (pos <= f) continue;
                double* wj = W + int64_t(j) * ldw;
                if (beta != 0.0) {
                    double sdot = 0.0;
                    for (int i = f + lane; i < m; i += 32) sdot += vsh[i] * wj[i];
                    const double fct = beta * warp_sum(sdot);
                    for (int i = f + lane; i < m; i += 32) wj[i] -= fct * vsh[i];
                    __syncwarp();
                }
                const double d = wj[f];
                double s2 = 0.0;
                if (cnS[j - j0] - d * d < 1e-6 * rnS[j - j0] || a.tol_mode) {
                    for (int i = f + 1 + lane; i < m; i += 32) s2 += wj[i] * wj[i];
                    s2 = warp_sum(s2);
                }
                downdate(j, pos, d, s2);
            }
        }
        mark(2);
        publish(bv, bp, tr);
        mark(3);
        if (spv >= j0 && spv < j1) {
            pend_s = spv;
            pend_f = f;
            pend_alpha = zero ? 0.0 : alpha;
        }
        ++frank;
        grid_sync(a.bar);
        mark(4);
        if (a.tol_mode && frank < a.rmax) {
            double tt = 0.0;
            for (int c = 0; c < G; ++c) tt += a.slot_t[par * G + c];
            const double r = sqrt(tt);
            if (g == 0 && t == 0) *a.res = r;
            if (r <= a.tol) reached = true;
        }
    }
    finish_pending();
    if (clk)
        for (int i = 0; i < 5; ++i) a.phase_clk[i] = ph[i];
    if (g == 0) {
        for (int i = t; i < n; i += blockDim.x) a.perm[i] = p2s[i];
        if (t == 0) {
            a.out[0] = frank;
            a.out[1] = reached ? 1 : 0;
        }
    }
}

// ------------------------------------------- resident columns (m <= 768) ---
// cpqr_step_kernel with every CTA's columns held ON CHIP for the whole
// factorization instead of re-read and re-written through L2 each step: two
// columns per warp in registers (row i at lane i % 32, slot i / 32) and the
// rest in shared memory.  The pivot column reaches the other CTAs through a
// per-CTA candidate slot: after its apply each CTA publishes its best
// candidate's value, position and storage index AND the column itself
// (slot_col), so after the step's one grid barrier every CTA forms H_f from
// the winner's published copy.  Positions live with the columns (no n-sized
// maps): the column at position f takes the pivot's old position, the pivot
// takes f.  Same reflector, downdate and tie-break rules as the other CPQR
// kernels (core/qr.hpp:140-236); only the summation order of the column dot
// products differs (fixed rows per lane).
constexpr int kResRegCols = 4;  // register-resident columns per warp
constexpr int kResRows = 20;    // rows per lane (m <= 640)
constexpr int kResThreads = 256;  // 8 warps: 4 x 20 + 20 doubles of registers per lane

__global__ void __launch_bounds__(kResThreads, 1) cpqr_res_kernel(CpqrArgs a) {
    extern __shared__ double rsm[];
    const int m = a.m, n = a.n;
    const int G = gridDim.x, g = blockIdx.x, t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31, nw = blockDim.x >> 5;
    const int cpb = (n + G - 1) / G;
    const int j0 = g * cpb, j1 = min(n, j0 + cpb), nown = max(0, j1 - j0);
    const int nreg = kResRegCols * nw;  // local columns [0, nreg) in registers
    const int UR = (m + 31) >> 5, MP = 32 * UR;  // row chunks; shared-memory column pitch (rows >= m zero)
    double* vsh = rsm;                   // m: H_f's vector
    double* cnS = vsh + m;               // cpb
    double* rnS = cnS + cpb;             // cpb
    double* colS = rnS + cpb;            // (cpb - nreg) x MP shared-memory columns
    int* posS = reinterpret_cast<int*>(colS + size_t(max(0, cpb - nreg)) * MP);  // cpb positions
    __shared__ double sv[32], st[32], shb[32];
    __shared__ int sp[32], ss[32];
    __shared__ int s_piv, s_spv, s_win, s_best_c;
    double xr[kResRegCols][kResRows];  // this warp's register columns
    auto lc_of = [&](int b) { return warp * kResRegCols + b; };  // local index of register column b
    const bool clk = a.phase_clk != nullptr && g == 0 && t == 0;
    long long ph[5] = {0, 0, 0, 0, 0}, c0 = clock64();
    auto mark = [&](int i) {
        if (clk) {
            const long long c1 = clock64();
            ph[i] += c1 - c0;
            c0 = c1;
        }
    };
    // ---- load the owned columns, initial positions
#pragma unroll
    for (int b = 0; b < kResRegCols; ++b) {
        const int c = lc_of(b);
#pragma unroll
        for (int u = 0; u < kResRows; ++u) {
            const int i = lane + 32 * u;
            xr[b][u] = (c < nown && i < m) ? a.W[i + int64_t(j0 + c) * a.ldw] : 0.0;
        }
    }
    for (int c = nreg; c < nown; ++c)
        for (int i = t; i < MP; i += blockDim.x) colS[size_t(c - nreg) * MP + i] = i < m ? a.W[i + int64_t(j0 + c) * a.ldw] : 0.0;
    for (int c = t; c < cpb; c += blockDim.x) posS[c] = j0 + c;
    __syncthreads();

    int par = 0;
    // CTA best (value desc, position asc) over the warps' bests, the slot
    // record, then the winning column's data into slot_col[par][g]
    auto publish = [&](double bv, int bp, int bc, double tr) {
        if (lane == 0) {
            sv[warp] = bv;
            sp[warp] = bp;
            ss[warp] = bc;
            st[warp] = tr;
        }
        __syncthreads();
        if (t == 0) {
            double v = -DBL_MAX, tt = 0.0;
            int p = INT_MAX, c = -1;
            for (int w = 0; w < nw; ++w) {
                if (better(sv[w], sp[w], v, p)) {
                    v = sv[w];
                    p = sp[w];
                    c = ss[w];
                }
                tt += st[w];
            }
            a.slot_v[par * G + g] = v;
            a.slot_p[par * G + g] = p;
            a.slot_s[par * G + g] = c >= 0 ? j0 + c : -1;
            a.slot_t[par * G + g] = tt;
            s_best_c = c;
        }
        __syncthreads();
        const int c = s_best_c;
        double* dst = a.slot_col + (size_t(par) * G + g) * m;
        if (c >= 0 && c < nreg) {
            if (warp == c / kResRegCols) {
#pragma unroll
                for (int b = 0; b < kResRegCols; ++b)
                    if (c == lc_of(b)) {
#pragma unroll
                        for (int u = 0; u < kResRows; ++u)
                            if (lane + 32 * u < m) __stcg(dst + lane + 32 * u, xr[b][u]);
                    }
            }
        } else if (c >= nreg) {
            for (int i = t; i < m; i += blockDim.x) __stcg(dst + i, colS[size_t(c - nreg) * MP + i]);
        }
    };

    // ---- squared norms (core/qr.hpp:157-161), fixed rows per lane
    {
        double bv = -DBL_MAX, tr = 0.0;
        int bp = INT_MAX, bc = -1;
        for (int c = nreg + warp; c < nown; c += nw) {  // shared-memory columns
            double sum = 0.0;
            for (int u = 0; u < kResRows; ++u) {
                const int i = lane + 32 * u;
                if (i < m) {
                    const double x = colS[size_t(c - nreg) * MP + i];
                    sum += x * x;
                }
            }
            sum = warp_sum(sum);
            if (lane == 0) {
                cnS[c] = sum;
                rnS[c] = sum;
            }
            if (better(sum, j0 + c, bv, bp)) {
                bv = sum;
                bp = j0 + c;
                bc = c;
            }
            tr += sum;
        }
#pragma unroll
        for (int b = 0; b < kResRegCols; ++b) {
            const int c = lc_of(b);
            double sum = 0.0;
#pragma unroll
            for (int u = 0; u < kResRows; ++u) sum += xr[b][u] * xr[b][u];
            sum = warp_sum(sum);
            if (c < nown) {
                if (lane == 0) {
                    cnS[c] = sum;
                    rnS[c] = sum;
                }
                if (better(sum, j0 + c, bv, bp)) {
                    bv = sum;
                    bp = j0 + c;
                    bc = c;
                }
                tr += sum;
            }
        }
        publish(bv, bp, bc, tr);
    }
    grid_sync(a.bar);

    int frank = 0;
    bool reached = false;
    if (a.tol_mode) {
        double tt = 0.0;
        for (int c = 0; c < G; ++c) tt += a.slot_t[c];
        const double r = sqrt(tt);
        reached = r <= a.tol;
        if (g == 0 && t == 0) *a.res = r;
    }
    int pend_c = -1, pend_f = 0;  // own pivot column whose rows pend_f.. become (alpha, 0, ...)
    double pend_alpha = 0.0;
    auto finish_pending = [&]() {
        if (pend_c < 0) return;
        if (pend_c < nreg) {
#pragma unroll
            for (int b = 0; b < kResRegCols; ++b)
                if (pend_c == lc_of(b)) {
#pragma unroll
                    for (int u = 0; u < kResRows; ++u) {
                        const int i = lane + 32 * u;
                        if (i >= pend_f) xr[b][u] = (i == pend_f) ? pend_alpha : 0.0;
                    }
                }
        } else {
            for (int i = pend_f + t; i < m; i += blockDim.x)
                colS[size_t(pend_c - nreg) * MP + i] = (i == pend_f) ? pend_alpha : 0.0;
        }
        pend_c = -1;
    };
    while (!reached && frank < a.kmax) {
        const int f = frank;
        finish_pending();
        // 1. pivot (value desc, position asc) over the CTA slots
        if (warp == 0) {
            double v = -DBL_MAX;
            int p = INT_MAX, c = -1;
            for (int q = lane; q < G; q += 32)
                if (better(a.slot_v[par * G + q], a.slot_p[par * G + q], v, p)) {
                    v = a.slot_v[par * G + q];
                    p = a.slot_p[par * G + q];
                    c = q;
                }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, v, o);
                const int op = __shfl_xor_sync(0xffffffffu, p, o);
                const int oc = __shfl_xor_sync(0xffffffffu, c, o);
                if (better(ov, op, v, p)) {
                    v = ov;
                    p = op;
                    c = oc;
                }
            }
            if (lane == 0) {
                s_piv = p;
                s_win = c;
                s_spv = a.slot_s[par * G + c];
            }
        }
        __syncthreads();
        const int piv = s_piv, spv = s_spv, win = s_win;
        mark(0);
        // 2. householder_step on the published pivot column (core/qr.hpp:44-66), in every CTA
        const double* pc = a.slot_col + (size_t(par) * G + win) * m;
        double sum = 0.0;
        for (int i = f + t; i < m; i += blockDim.x) {
            const double x = __ldcg(pc + i);
            vsh[i] = x;
            sum += x * x;
        }
        sum = warp_sum(sum);
        if (lane == 0) shb[warp] = sum;
        __syncthreads();
        double norm2 = 0.0;
        for (int w = 0; w < nw; ++w) norm2 += shb[w];
        const double x1 = vsh[f];
        const double norm = sqrt(norm2);
        const bool zero = norm < 1e-300;
        const double alpha = x1 >= 0.0 ? -norm : norm;
        const double beta = zero ? 0.0 : 2.0 / (2.0 * (norm2 - alpha * x1));
        __syncthreads();
        if (zero) {
            for (int i = f + t; i < m; i += blockDim.x) vsh[i] = 0.0;
        } else if (t == 0) {
            vsh[f] = x1 - alpha;
        }
        // the swap (core/qr.hpp:182-187), on the owned positions
        for (int c = t; c < nown; c += blockDim.x) {
            const int pc_ = posS[c];
            posS[c] = (j0 + c == spv) ? f : (pc_ == f ? piv : pc_);
        }
        __syncthreads();
        if (g == 0) {
            for (int i = t; i < m; i += blockDim.x) a.Vst[i + int64_t(f) * m] = i < f ? 0.0 : vsh[i];
            if (t == 0) {
                a.beta[f] = beta;
                if (zero) a.out[2] = 1;
            }
        }
        mark(1);
        par ^= 1;  // this step's candidates go to the other buffer
        // 3. apply H_f to the own trailing columns, downdate (core/qr.hpp:190-200)
        // v(i) for this lane's rows, zero outside [f, m)
        double vr[kResRows];
#pragma unroll
        for (int u = 0; u < kResRows; ++u) {
            const int i = lane + 32 * u;
            vr[u] = (i >= f && i < m) ? vsh[i] : 0.0;
        }
        double bv = -DBL_MAX, tr = 0.0;
        int bp = INT_MAX, bc = -1;
        const int uf = f >> 5, lf = f & 31;
        // the downdate (core/qr.hpp:193-200) of local column c, whose row-f
        // entry is d and rows > f give s2 on demand; the warp's best candidate
        auto downdate = [&](int c, int pos, double d, auto&& tail_sq) {
            double c2 = cnS[c] - d * d;
            const double ref = rnS[c];
            double rr = ref;
            if (c2 < 1e-6 * ref || a.tol_mode) {  // uniform across the warp
                const double s2 = warp_sum(tail_sq());
                if (c2 < 1e-6 * ref) {
                    c2 = s2;
                    rr = s2;
                }
                tr += s2;
            }
            __syncwarp();
            if (lane == 0) {
                cnS[c] = c2;
                rnS[c] = rr;
            }
            __syncwarp();
            if (better(c2, pos, bv, bp)) {
                bv = c2;
                bp = pos;
                bc = c;
            }
        };
        // register columns: the warp's kResRegCols columns together (independent
        // dot-product chains and shuffle reductions interleave)
        {
            bool on[kResRegCols];
            int pos[kResRegCols];
#pragma unroll
            for (int b = 0; b < kResRegCols; ++b) {
                const int c = lc_of(b);
                pos[b] = c < nown ? posS[c] : -1;
                on[b] = c < nown && pos[b] > f;
            }
            if (beta != 0.0) {
                double sd[kResRegCols];
#pragma unroll
                for (int b = 0; b < kResRegCols; ++b) sd[b] = 0.0;
#pragma unroll
                for (int u = 0; u < kResRows; ++u)
#pragma unroll
                    for (int b = 0; b < kResRegCols; ++b) sd[b] += vr[u] * xr[b][u];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                    for (int b = 0; b < kResRegCols; ++b) sd[b] += __shfl_xor_sync(0xffffffffu, sd[b], o);
#pragma unroll
                for (int b = 0; b < kResRegCols; ++b) {
                    const double fct = on[b] ? beta * sd[b] : 0.0;
#pragma unroll
                    for (int u = 0; u < kResRows; ++u) xr[b][u] -= fct * vr[u];
                }
            }
#pragma unroll
            for (int b = 0; b < kResRegCols; ++b) {
                if (!on[b]) continue;
                double xf = 0.0;
#pragma unroll
                for (int u = 0; u < kResRows; ++u) xf = (u == uf) ? xr[b][u] : xf;
                const double d = __shfl_sync(0xffffffffu, xf, lf);  // row f
                downdate(lc_of(b), pos[b], d, [&] {
                    double s2 = 0.0;
#pragma unroll
                    for (int u = 0; u < kResRows; ++u) {
                        const int i = lane + 32 * u;
                        if (i > f && i < m) s2 += xr[b][u] * xr[b][u];
                    }
                    return s2;
                });
            }
        }
        // shared-memory columns, two at a time, updated in place
        for (int c0 = nreg + warp; c0 < nown; c0 += 2 * nw) {
            const int cc[2] = {c0, c0 + nw};
            bool on[2];
            int pos[2];
            double* col[2];
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                pos[b] = cc[b] < nown ? posS[cc[b]] : -1;
                on[b] = cc[b] < nown && pos[b] > f;
                col[b] = colS + size_t((on[b] ? cc[b] : nreg) - nreg) * MP;
            }
            if (!on[0] && !on[1]) continue;
            if (beta != 0.0) {
                // no row predicates: v is zero outside [f, m) and the padded
                // rows are zero, so rows < f add +-0 to the dot products and
                // keep their bits in the update — the same sums and values as
                // restricting to [f, m); only the warp-uniform chunk bound UR
                double sd[2] = {0.0, 0.0};
                const double* p0 = col[0] + lane;
                const double* p1 = col[1] + lane;
#pragma unroll
                for (int u = 0; u < kResRows; ++u)
                    if (u < UR) {
                        sd[0] += vr[u] * p0[32 * u];
                        sd[1] += vr[u] * p1[32 * u];
                    }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                    for (int b = 0; b < 2; ++b) sd[b] += __shfl_xor_sync(0xffffffffu, sd[b], o);
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    if (!on[b]) continue;
                    const double fct = beta * sd[b];
                    double* pb = col[b] + lane;
#pragma unroll
                    for (int u = 0; u < kResRows; ++u)
                        if (u < UR) pb[32 * u] -= fct * vr[u];
                }
                __syncwarp();
            }
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                if (!on[b]) continue;
                const double* cb = col[b];
                downdate(cc[b], pos[b], cb[f], [&] {
                    double s2 = 0.0;
                    for (int i = f + 1 + lane; i < m; i += 32) s2 += cb[i] * cb[i];
                    return s2;
                });
            }
        }
        mark(2);
        publish(bv, bp, bc, tr);
        mark(3);
        if (spv >= j0 && spv < j1) {
            pend_c = spv - j0;
            pend_f = f;
            pend_alpha = zero ? 0.0 : alpha;
        }
        ++frank;
        grid_sync(a.bar);
        mark(4);
        if (a.tol_mode && frank < a.rmax) {
            double tt = 0.0;
            for (int c = 0; c < G; ++c) tt += a.slot_t[par * G + c];
            const double r = sqrt(tt);
            if (g == 0 && t == 0) *a.res = r;
            if (r <= a.tol) reached = true;
        }
    }
    finish_pending();
    __syncthreads();
    if (clk)
        for (int i = 0; i < 5; ++i) a.phase_clk[i] = ph[i];
    // write the owned columns back (storage order) and their positions
#pragma unroll
    for (int b = 0; b < kResRegCols; ++b) {
        const int c = lc_of(b);
        if (c < nown) {
#pragma unroll
            for (int u = 0; u < kResRows; ++u) {
                const int i = lane + 32 * u;
                if (i < m) a.W[i + int64_t(j0 + c) * a.ldw] = xr[b][u];
            }
        }
    }
    for (int c = nreg; c < nown; ++c)
        for (int i = t; i < m; i += blockDim.x) a.W[i + int64_t(j0 + c) * a.ldw] = colS[size_t(c - nreg) * MP + i];
    for (int c = t; c < nown; c += blockDim.x) a.perm[posS[c]] = j0 + c;
    if (g == 0 && t == 0) {
        a.out[0] = frank;
        a.out[1] = reached ? 1 : 0;
    }
}

// Wp(:, p) = W(:, perm[p]): storage order -> position order
__global__ void gather_cols_kernel(const double* W, int64_t ldw, int m, int n, const int* perm, double* Wp,
                                   int64_t ldp) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(m) * n;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int j = int(e / m), i = int(e % m);
        Wp[i + int64_t(j) * ldp] = W[i + int64_t(perm[j]) * ldw];
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
// B and T may alias (each warp reads its whole column before writing it).
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

// T (nb x nc, in place) <- S^{-1} T for an upper-triangular nb x nb block, nb
// <= 64: S staged once per CTA in shared memory, one warp per right-hand side
// with its column in registers (lane owns rows lane, lane + 32), the pivots
// as reciprocals (the verified V = R^{-1} W solve; the ID's tri-solve keeps
// trisolve_kernel's division, the reference's arithmetic)
__global__ void __launch_bounds__(256) trisolve_reg_kernel(const double* S, int64_t lds, int nb, double* T,
                                                           int64_t ldt, int nc) {
    __shared__ double Ss[64][65];
    __shared__ double rp[64];
    for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
        const int i = e % 64, j = e / 64;
        Ss[i][j] = (i < nb && j < nb && i <= j) ? S[i + int64_t(j) * lds] : 0.0;
    }
    for (int i = threadIdx.x; i < 64; i += blockDim.x) rp[i] = i < nb ? 1.0 / S[i + int64_t(i) * lds] : 0.0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    for (int c = blockIdx.x * wpb + warp; c < nc; c += gridDim.x * wpb) {
        double* col = T + int64_t(c) * ldt;
        double b0 = lane < nb ? col[lane] : 0.0, b1 = lane + 32 < nb ? col[lane + 32] : 0.0;
        for (int i = nb - 1; i >= 0; --i) {
            const double xi = __shfl_sync(0xffffffffu, i < 32 ? b0 : b1, i & 31) * rp[i];
            if (lane == (i & 31)) {
                if (i < 32) b0 = xi;
                else b1 = xi;
            }
            if (lane < i) b0 -= Ss[lane][i] * xi;
            if (lane + 32 < i) b1 -= Ss[lane + 32][i] * xi;
        }
        if (lane < nb) col[lane] = b0;
        if (lane + 32 < nb) col[lane + 32] = b1;
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
    // one-barrier-per-step kernel when its shared maps fit (m + n <= 27k);
    // RLRA_CPQR_TWO_BARRIER=1 forces the two-barrier kernel
    static const bool two_bar = std::getenv("RLRA_CPQR_TWO_BARRIER") != nullptr;
    const int cpb_max = ceil_div(n, std::max(1, std::min(ctx.num_sms, ceil_div(n, 4 * (kCpqrThreads / 32)))));
    const size_t step_smem = sizeof(double) * (size_t(m) + 2 * size_t(cpb_max)) + 2 * sizeof(int) * size_t(n);
    bool one_bar = !two_bar && step_smem <= 220 * 1024;
    int per_sm = 0;
    if (one_bar) {
        RLRA_CUDA(cudaFuncSetAttribute(cpqr_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(step_smem)));
        RLRA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cpqr_step_kernel, kCpqrStepThreads, step_smem));
        one_bar = per_sm >= 1;
    }
    if (!one_bar)
        RLRA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cpqr_coop_kernel, kCpqrThreads, 0));
    int G = std::max(1, std::min(ctx.num_sms * std::max(1, per_sm), ceil_div(n, 4 * (kCpqrThreads / 32))));
    G = std::min(G, ctx.num_sms);
    // resident-columns kernel when every CTA's columns fit on chip (two per
    // warp in registers, the rest in shared memory) and m <= 32 * kCpqrRegs;
    // RLRA_CPQR_RESIDENT=0 keeps the streaming kernel
    static const bool res_env = !(std::getenv("RLRA_CPQR_RESIDENT") && std::getenv("RLRA_CPQR_RESIDENT")[0] == '0');
    const int Gr = std::min(ctx.num_sms, std::max(1, n));
    const int cpb_r = ceil_div(n, Gr), nreg_r = kResRegCols * (kResThreads / 32);
    const size_t res_smem = sizeof(double) * (size_t(m) + 2 * size_t(cpb_r) +
                                              size_t(std::max(0, cpb_r - nreg_r)) * size_t(32 * ceil_div(m, 32))) +
                            sizeof(int) * size_t(cpb_r);
    bool resident = res_env && !two_bar && m <= 32 * kResRows && res_smem <= 224 * 1024;
    if (resident) {
        RLRA_CUDA(cudaFuncSetAttribute(cpqr_res_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(res_smem)));
        int per = 0;
        RLRA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, cpqr_res_kernel, kResThreads, res_smem));
        resident = per >= 1;
        if (resident) {
            G = Gr;
            one_bar = true;
        }
    }
    Buf sv(ctx, sizeof(double) * 2 * G), sp(ctx, sizeof(int) * 2 * G), stt(ctx, sizeof(double) * 2 * G),
        sst(ctx, sizeof(int) * 2 * G), scol(ctx, resident ? sizeof(double) * 2 * size_t(G) * m : 8);
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
    static const bool want_clk = std::getenv("RLRA_CPQR_PHASES") != nullptr;
    Buf clkb(ctx, sizeof(long long) * 8);
    a.phase_clk = (want_clk && one_bar) ? reinterpret_cast<long long*>(clkb.p) : nullptr;
    a.slot_s = sst.i();
    a.slot_col = scol.d();
    void* args[] = {&a};
    if (resident) {
        RLRA_CUDA(cudaLaunchCooperativeKernel((void*)cpqr_res_kernel, dim3(G), dim3(kResThreads), args, res_smem,
                                              ctx.stream));
    } else if (one_bar) {
        RLRA_CUDA(cudaLaunchCooperativeKernel((void*)cpqr_step_kernel, dim3(G), dim3(kCpqrStepThreads), args,
                                              step_smem, ctx.stream));
    } else {
        RLRA_CUDA(cudaLaunchCooperativeKernel((void*)cpqr_coop_kernel, dim3(G), dim3(kCpqrThreads), args,
                                              0, ctx.stream));
    }
    ++ctx.launches;
    if (a.phase_clk) {
        long long h[5];
        RLRA_CUDA(cudaMemcpyAsync(h, clkb.p, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
        RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
        std::fprintf(stderr, "cpqr_step m=%d n=%d G=%d clocks: pivot %lld householder %lld apply %lld publish %lld sync %lld\n",
                     m, n, G, h[0], h[1], h[2], h[3], h[4]);
    }
    if (one_bar) {  // storage order -> position order
        DMatBuf Wp(ctx, m, n);
        const int blocks = int(std::min<int64_t>((int64_t(m) * n + 255) / 256, int64_t(ctx.num_sms) * 8));
        gather_cols_kernel<<<blocks, 256, 0, ctx.stream>>>(W.m.p, W.m.ld, m, n, perm, Wp.m.p, Wp.m.ld);
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
        std::swap(W, Wp);
    }
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

void upper_tri_solve_inplace(Context& ctx, const DMat& S11, const DMat& T, bool fast) {
    // Blocked back substitution on DMMA: for the diagonal blocks from the
    // bottom up, T_I <- S_II^{-1} T_I (one warp per right-hand side, the
    // block's column in shared memory), then the rank-kTriNB update
    // T[0:i0, :] -= S[0:i0, I] T_I on the tensor-core GEMM.  Shared memory
    // holds one kTriNB slice per warp, so k is unbounded; the
    // contraction's k^2 (n - k) flops run on DMMA.
    const int k = int(S11.rows), nc = int(T.cols);
    if (k == 0 || nc == 0) return;
    constexpr int kTriNB = 64, kWpb = 8, kTriRec = 512;
    if (k > kTriRec) {
        // recursive halving (split on a kTriNB boundary): T2 <- S22^{-1} T2,
        // T1 -= S12 T2 with K = k2 >= 256 (the rank-64 updates of the flat loop
        // ran at ~8 TFLOP/s), T1 <- S11^{-1} T1
        const int k1 = ((k / 2 + kTriNB - 1) / kTriNB) * kTriNB, k2 = k - k1;
        upper_tri_solve_inplace(ctx, S11.block(k1, k1, k2, k2), T.block(k1, 0, k2, nc), fast);
        gemm(ctx, Op::N, Op::N, -1.0, S11.block(0, k1, k1, k2), T.block(k1, 0, k2, nc), 1.0, T.block(0, 0, k1, nc));
        upper_tri_solve_inplace(ctx, S11.block(0, 0, k1, k1), T.block(0, 0, k1, nc), fast);
        return;
    }
    const size_t smem = sizeof(double) * size_t(kTriNB) * kWpb;
    const int blocks = std::max(1, std::min(ctx.num_sms * 4, ceil_div(nc, kWpb)));
    for (int i0 = ((k - 1) / kTriNB) * kTriNB; i0 >= 0; i0 -= kTriNB) {  // block rows aligned at 0
        const int nb = std::min(k, i0 + kTriNB) - i0;
        if (fast)
            trisolve_reg_kernel<<<blocks, kWpb * 32, 0, ctx.stream>>>(S11.p + i0 + int64_t(i0) * S11.ld, S11.ld, nb,
                                                                     T.p + i0, T.ld, nc);
        else
            trisolve_kernel<<<blocks, kWpb * 32, smem, ctx.stream>>>(S11.p + i0 + int64_t(i0) * S11.ld, S11.ld, nb,
                                                                     T.p + i0, T.ld, nc, T.p + i0, T.ld);
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
        if (i0 > 0)
            gemm(ctx, Op::N, Op::N, -1.0, S11.block(0, i0, i0, nb), T.block(i0, 0, nb, nc), 1.0,
                 T.block(0, 0, i0, nc));
    }
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
        copy_mat(ctx, S12, T);
        upper_tri_solve_inplace(ctx, S11, T);
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
