// jacobi.cu — one-sided Jacobi SVD and two-sided Jacobi eigensolver.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <unistd.h>
#include <cstring>
#include <string>

#include "cpqr.cuh"
#include "gemm.cuh"
#include "jacobi.cuh"
#include "reduce.cuh"

namespace cg = cooperative_groups;

namespace rlra_b200 {

namespace {

constexpr int kJacThreads = 256;
constexpr int kJacReg = 16;  // register-resident column slice per lane (m <= 512)
constexpr int kOneSidedSweepCap = 60;  // reference core/jacobi.hpp:29
constexpr int kTwoSidedSweepCap = 30;  // reference core/jacobi.hpp:28

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// column at tournament position `pos` in round r (position 0 is fixed)
__device__ __forceinline__ int rr_col(int pos, int r, int n2) {
    return pos == 0 ? 0 : ((pos - 1 + r) % (n2 - 1)) + 1;
}

struct OneSidedArgs {
    unsigned* bar;  // grid_sync state (Context::gbar)
    double* W;
    int64_t ldw;
    int m, n;
    double* V;
    int64_t ldv;
    int* flags;   // [0..2] rotated-in-sweep flags, [3] status, [4] sweeps used
};

__global__ void __launch_bounds__(kJacThreads) onesided_jacobi_kernel(OneSidedArgs a) {
    const int n = a.n, m = a.m;
    const int n2 = n + (n & 1);
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const double eps = 1e-15;  // reference core/jacobi.hpp:156
    volatile int* flags = a.flags;
    int sweep = 0;
    for (;;) {
        if (sweep >= kOneSidedSweepCap) {
            if (blockIdx.x == 0 && threadIdx.x == 0) flags[3] = RLRA_ECONV;
            break;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) flags[(sweep + 1) % 3] = 0;
        for (int r = 0; r < n2 - 1; ++r) {
            for (int pi = gw; pi < n2 / 2; pi += nw) {
                const int ca = rr_col(pi, r, n2), cb = rr_col(n2 - 1 - pi, r, n2);
                const int p = min(ca, cb), q = max(ca, cb);
                if (q >= n) continue;
                double* wp = a.W + int64_t(p) * a.ldw;
                double* wq = a.W + int64_t(q) * a.ldw;
                double app = 0.0, aqq = 0.0, apq = 0.0;
                for (int i = lane; i < m; i += 32) {
                    const double xp = wp[i], xq = wq[i];
                    app += xp * xp;
                    aqq += xq * xq;
                    apq += xp * xq;
                }
                app = warp_sum(app);
                aqq = warp_sum(aqq);
                apq = warp_sum(apq);
                if (app == 0.0 || aqq == 0.0) continue;
                if (fabs(apq) <= eps * sqrt(app * aqq)) continue;
                const double zeta = (aqq - app) / (2.0 * apq);
                const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double s = t * c;
                for (int i = lane; i < m; i += 32) {
                    const double xp = wp[i], xq = wq[i];
                    wp[i] = c * xp - s * xq;
                    wq[i] = s * xp + c * xq;
                }
                double* vp = a.V + int64_t(p) * a.ldv;
                double* vq = a.V + int64_t(q) * a.ldv;
                for (int i = lane; i < n; i += 32) {
                    const double xp = vp[i], xq = vq[i];
                    vp[i] = c * xp - s * xq;
                    vq[i] = s * xp + c * xq;
                }
                if (lane == 0) flags[sweep % 3] = 1;
            }
            grid_sync(a.bar);
        }
        const int rotated = flags[sweep % 3];
        ++sweep;
        if (!rotated || n < 2) break;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) flags[4] = sweep;
}

// ------------------------------------------------ block one-sided Jacobi ---
// Columns are grouped into blocks of BW.  In each outer round every CTA takes
// one block pair (I, J) from a round-robin tournament over the blocks, stages
// the 2*BW columns of W in shared memory, runs one pass of the reference's
// pairwise rotations over all column pairs inside the pair (an inner
// round-robin, one warp per pair), writes the columns back and applies the
// accumulated 2BW x 2BW rotation to the same columns of V.  One grid barrier
// per outer round instead of one per column round; the rotation formula, the
// skip rule and the "sweep without rotations" stop are the reference's
// (core/jacobi.hpp:164-199).
struct BlockJacArgs {
    unsigned* bar;  // grid_sync state (Context::gbar)
    double* W;
    int64_t ldw;
    int m, n;
    double* V;
    int64_t ldv;
    int nb;       // number of blocks (even)
    int* flags;   // [0..2] rotated-in-sweep, [3] status, [4] sweeps used
};

template <int BW>
__global__ void __launch_bounds__(BW * 32) block_jacobi_kernel(BlockJacArgs a) {
    constexpr int C2 = 2 * BW;
    extern __shared__ double bj_smem[];
    double* Ws = bj_smem;                      // C2 columns of length m
    double* Jm = bj_smem + size_t(C2) * a.m;   // C2 x C2 accumulated rotation
    __shared__ int s_rot;
    const int m = a.m, n = a.n, nb = a.nb;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x;
    const double eps = 1e-15;
    volatile int* flags = a.flags;
    int sweep = 0;
    for (;;) {
        if (sweep >= kOneSidedSweepCap) {
            if (g == 0 && threadIdx.x == 0) flags[3] = RLRA_ECONV;
            break;
        }
        if (g == 0 && threadIdx.x == 0) flags[(sweep + 1) % 3] = 0;
        for (int r = 0; r < nb - 1; ++r) {
            const int b1 = rr_col(g, r, nb), b2 = rr_col(nb - 1 - g, r, nb);
            const int bI = min(b1, b2), bJ = max(b1, b2);
            auto gcol = [&](int c) { return c < BW ? bI * BW + c : bJ * BW + (c - BW); };
            // stage W columns (zero-padded past n) and reset the rotation
            // cp.async so all of a column's loads are in flight at once
            // (a load-then-store loop would serialise on L2 latency)
            for (int c = warp; c < C2; c += BW) {
                const int gc = gcol(c);
                double* dst = Ws + size_t(c) * m;
                if (gc < n) {
                    const double* src = a.W + int64_t(gc) * a.ldw;
                    for (int i = lane; i < m; i += 32) {
                        const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst + i));
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src + i));
                    }
                } else {
                    for (int i = lane; i < m; i += 32) dst[i] = 0.0;
                }
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
            for (int e = threadIdx.x; e < C2 * C2; e += blockDim.x) Jm[e] = (e % C2 == e / C2) ? 1.0 : 0.0;
            if (threadIdx.x == 0) s_rot = 0;
            __syncthreads();
            for (int ir = 0; ir < C2 - 1; ++ir) {
                const int c1 = rr_col(warp, ir, C2), c2 = rr_col(C2 - 1 - warp, ir, C2);
                const int p = min(c1, c2), q = max(c1, c2);
                if (gcol(q) < n) {
                    double* wp = Ws + size_t(p) * m;
                    double* wq = Ws + size_t(q) * m;
                    double app = 0.0, aqq = 0.0, apq = 0.0;
                    // columns up to 32 * kJacReg long stay in registers between
                    // the dot products and the rotation (loads issued together)
                    const bool regs = m <= 32 * kJacReg;
                    double rp[kJacReg], rq[kJacReg];
                    if (regs) {
#pragma unroll
                        for (int u = 0; u < kJacReg; ++u) {
                            const int i = lane + 32 * u;
                            rp[u] = i < m ? wp[i] : 0.0;
                            rq[u] = i < m ? wq[i] : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < kJacReg; ++u) {
                            app += rp[u] * rp[u];
                            aqq += rq[u] * rq[u];
                            apq += rp[u] * rq[u];
                        }
                    } else {
                        for (int i = lane; i < m; i += 32) {
                            const double xp = wp[i], xq = wq[i];
                            app += xp * xp;
                            aqq += xq * xq;
                            apq += xp * xq;
                        }
                    }
                    app = warp_sum(app);
                    aqq = warp_sum(aqq);
                    apq = warp_sum(apq);
                    if (app != 0.0 && aqq != 0.0 && fabs(apq) > eps * sqrt(app * aqq)) {
                        const double zeta = (aqq - app) / (2.0 * apq);
                        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                        const double c = rsqrt(1.0 + t * t);
                        const double s = t * c;
                        if (regs) {
#pragma unroll
                            for (int u = 0; u < kJacReg; ++u) {
                                const int i = lane + 32 * u;
                                if (i < m) {
                                    wp[i] = c * rp[u] - s * rq[u];
                                    wq[i] = s * rp[u] + c * rq[u];
                                }
                            }
                        } else {
                            for (int i = lane; i < m; i += 32) {
                                const double xp = wp[i], xq = wq[i];
                                wp[i] = c * xp - s * xq;
                                wq[i] = s * xp + c * xq;
                            }
                        }
                        if (lane < C2) {
                            const double xp = Jm[p * C2 + lane], xq = Jm[q * C2 + lane];
                            Jm[p * C2 + lane] = c * xp - s * xq;
                            Jm[q * C2 + lane] = s * xp + c * xq;
                        }
                        if (lane == 0) s_rot = 1;
                    }
                }
                __syncthreads();
            }
            if (s_rot) {
                for (int c = warp; c < C2; c += BW) {
                    const int gc = gcol(c);
                    if (gc < n)
                        for (int i = lane; i < m; i += 32) a.W[i + int64_t(gc) * a.ldw] = Ws[size_t(c) * m + i];
                }
                // V(:, cols) <- V(:, cols) * Jm, one row per thread
                for (int i = threadIdx.x; i < n; i += blockDim.x) {
                    double x[C2];
#pragma unroll
                    for (int c = 0; c < C2; ++c) {
                        const int gc = gcol(c);
                        x[c] = gc < n ? a.V[i + int64_t(gc) * a.ldv] : 0.0;
                    }
                    // row i is read completely before any of it is written
#pragma unroll
                    for (int c = 0; c < C2; ++c) {
                        double s = 0.0;
#pragma unroll
                        for (int t = 0; t < C2; ++t) s += x[t] * Jm[c * C2 + t];
                        const int gc = gcol(c);
                        if (gc < n) a.V[i + int64_t(gc) * a.ldv] = s;
                    }
                }
                if (threadIdx.x == 0) flags[sweep % 3] = 1;
            }
            grid_sync(a.bar);
        }
        const int rotated = flags[sweep % 3];
        ++sweep;
        if (!rotated || n < 2) break;
    }
    if (g == 0 && threadIdx.x == 0) flags[4] = sweep;
}

// sigma_j = ||W(:,j)||, one warp per column (fixed order)
__global__ void colnorm_kernel(const double* W, int64_t ldw, int m, int n, double* out) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int j = gw; j < n; j += nw) {
        double s = 0.0;
        for (int i = lane; i < m; i += 32) {
            const double x = W[i + int64_t(j) * ldw];
            s += x * x;
        }
        s = warp_sum(s);
        if (lane == 0) out[j] = sqrt(s);
    }
}

// stable descending rank of each key (std::stable_sort with '>')
__global__ void rank_desc_kernel(const double* key, int n, int* rank) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const double kj = key[j];
        int r = 0;
        for (int i = 0; i < n; ++i) {
            const double ki = key[i];
            r += (ki > kj) || (ki == kj && i < j);
        }
        rank[j] = r;
    }
}

// U(:, rank_j) = W(:, j)/sigma_j, V_out(:, rank_j) = V(:, j), sigma_out[rank_j]
__global__ void svd_scatter_kernel(const double* W, int64_t ldw, int m, int n, const double* V,
                                   int64_t ldv, int vrows, const double* sg, const int* rank,
                                   double* U, int64_t ldu, double* Vo, int64_t ldvo,
                                   double* sigma_out, int* needs) {
    const int64_t tot = int64_t(max(m, vrows)) * n;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int j = int(e / max(m, vrows)), i = int(e % max(m, vrows));
        const int r = rank[j];
        const double s = sg[j];
        if (i < m) U[i + int64_t(r) * ldu] = s > 1e-300 ? W[i + int64_t(j) * ldw] / s : 0.0;
        if (i < vrows) Vo[i + int64_t(r) * ldvo] = V[i + int64_t(j) * ldv];
        if (i == 0) {
            sigma_out[r] = s > 1e-300 ? s : 0.0;
            needs[r] = s > 1e-300 ? 0 : 1;
        }
    }
}

__device__ double block_sum_fixed(double v, double* sh) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) t += sh[i];
    __syncthreads();
    return t;
}

// Orthonormal completion for sigma == 0 columns (reference jacobi.hpp:33-60),
// one CTA, sequential over the columns that need it.  `done` scratch has n
// ints, r scratch has m doubles.
__global__ void completion_kernel(double* U, int64_t ldu, int m, int n, const int* needs, int* done,
                                  double* r) {
    __shared__ double sh[32];
    __shared__ double sv[32];
    __shared__ int si[32];
    __shared__ int nd;
    // the common case — no column needs completion — leaves at once
    int any = 0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) any |= needs[j];
    if (!__syncthreads_or(any)) return;
    if (threadIdx.x == 0) {
        nd = 0;
        for (int j = 0; j < n; ++j)
            if (!needs[j]) done[nd++] = j;
    }
    __syncthreads();
    for (int j = 0; j < n; ++j) {
        if (!needs[j]) continue;
        // best axis: smallest presence in the spanned set, first index wins
        double bv = -2.0;
        int bi = 0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            double proj2 = 0.0;
            for (int c = 0; c < nd; ++c) {
                const double u = U[i + int64_t(done[c]) * ldu];
                proj2 += u * u;
            }
            const double res = 1.0 - proj2;
            if (res > bv) {
                bv = res;
                bi = i;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if ((threadIdx.x & 31) == 0) {
            sv[threadIdx.x >> 5] = bv;
            si[threadIdx.x >> 5] = bi;
        }
        __syncthreads();
        int best = si[0];
        double bestv = sv[0];
        for (int w = 1; w < int(blockDim.x >> 5); ++w)
            if (sv[w] > bestv || (sv[w] == bestv && si[w] < best)) {
                bestv = sv[w];
                best = si[w];
            }
        for (int i = threadIdx.x; i < m; i += blockDim.x) r[i] = (i == best) ? 1.0 : 0.0;
        __syncthreads();
        for (int pass = 0; pass < 2; ++pass) {
            for (int c = 0; c < nd; ++c) {
                const double* uc = U + int64_t(done[c]) * ldu;
                double s = 0.0;
                for (int i = threadIdx.x; i < m; i += blockDim.x) s += uc[i] * r[i];
                const double dot = block_sum_fixed(s, sh);
                for (int i = threadIdx.x; i < m; i += blockDim.x) r[i] -= dot * uc[i];
                __syncthreads();
            }
        }
        double s = 0.0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) s += r[i] * r[i];
        const double nrm = sqrt(block_sum_fixed(s, sh));
        for (int i = threadIdx.x; i < m; i += blockDim.x) U[i + int64_t(j) * ldu] = r[i] / nrm;
        __syncthreads();
        if (threadIdx.x == 0) done[nd++] = j;
        __syncthreads();
    }
}

// ------------------------------------ Gram block one-sided Jacobi (large m) ---
// For inputs whose column pairs do not fit shared memory (the C2 R-hat is
// 6100 x 6100): columns in blocks of kGB; each outer round one CTA per block
// pair (I, J) (round-robin tournament over the blocks):
//   1. G = W_p^T W_p (64 x 64) streamed over the rows (DMMA, 8 warps of 16x32);
//   2. inner cyclic Jacobi sweeps on G, the reference rotation formula and
//      skip rule applied to (G_pp, G_qq, G_pq) — the same dot products the
//      reference's one-sided sweep forms — accumulating J (64 x 64);
//   3. W_p <- W_p J and V_p <- V_p J (streamed row chunks, DMMA).
// One grid barrier per outer round; a sweep with no rotation in any pair
// stops (reference core/jacobi.hpp:164-199 stop rule, on fresh Grams).
constexpr int kGB = 32;
constexpr int kGP = 2 * kGB;
constexpr int kGPitch = kGP + 1;
constexpr int kGChunk = 32;
constexpr int kGCP = kGChunk + 4;   // chunk pitch: m8n8k4 fragment loads conflict-free
constexpr int kGJP = kGP + 4;       // J copy for the DMMA apply, same reason
constexpr int kGInnerCap = 1;  // one inner sweep per visit: fastest overall (C2: 1 -> 3.0 s, 3 -> 3.7 s)
constexpr size_t kGramJacSmem = sizeof(double) * (2 * kGP * kGPitch + kGP * kGCP + kGP * kGJP);

__device__ __forceinline__ void jac_dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

struct GramJacArgs {
    unsigned* bar;
    double* W;
    int64_t ldw;
    int m, n;
    double* V;
    int64_t ldv;
    int nb;      // column blocks (even)
    int* flags;  // [0..2] rotated-in-sweep, [3] status, [4] sweeps used
    int inner_cap;
    long long* phase_clk;  // optional: CTA 0's clock64 per phase (RLRA_JACOBI_PHASES)
    unsigned* ver;         // bgram: block versions + J hand-off flags (zeroed; see the kernel)
    double* jbuf;          // bgram with helpers: 2 J slots per pair
    int helpers;           // bgram: V helper CTAs (grid = nb)
    // sgram: exact skip of clean pairs (zeroed per call; see sgram_jacobi_kernel)
    unsigned* mod;                 // [nb] stamp of the block's last modification
    unsigned* clean;               // [nb * nb + nb / 2] stamp of the pair's last rotation-free visit
    unsigned long long* counters;  // [0] visits, [1] skipped, [2] rotating
    // sgram: V updates ordered apart from W (zeroed per call): vtick[b] = V
    // updates of block b handed out (advanced by the W-chain owner),
    // vdone[b] = V updates of block b completed
    unsigned* vtick;
    unsigned* vdone;
    unsigned* tasks;  // sgram: [sweep cap] visit counters (zeroed per call)
    int skip_v;       // sgram: rotate W only (V recovered afterwards as R^{-1} W, see small_svd_tall)
    // sgram, W only: each visit split into two row halves taken as separate
    // tasks (2 CTAs per pair), partial Grams exchanged through xg
    int halves;
    double* xg;       // [2 generations][np slots][2 halves][kSXG] partial Grams (upper triangle)
    unsigned* xstamp; // [2 np][2]: partial of round R written (R + 1)
    unsigned* xack;   // [2 np][2]: partner's partial of round R read (R + 1)
    volatile unsigned* dbg;  // RLRA_SGRAM_DEBUG: mapped host record of a wait that timed out (then trap)
};


// ---- bulk-copy / mbarrier / release-acquire helpers (bgram staging) ----
__device__ __forceinline__ unsigned jb_smem(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void jb_bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(jb_smem(dst)),
        "l"(src), "r"(bytes), "r"(jb_smem(bar))
        : "memory");
}
__device__ __forceinline__ void jb_mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(jb_smem(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void jb_wait_at_least(const unsigned* p, unsigned v) {
    unsigned cur, ns = 32;
    for (;;) {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(p) : "memory");
        if (cur >= v) break;
        __nanosleep(ns);
        ns = ns < 128 ? ns * 2 : 128;
    }
}

// a version/stamp wait that, in debug mode, records itself and traps after ~1 s
__device__ __forceinline__ void sg_wait_dbg(const unsigned* p, unsigned v, volatile unsigned* dbg, unsigned code,
                                            unsigned R, unsigned hh) {
    if (!dbg) {
        jb_wait_at_least(p, v);
        return;
    }
    unsigned cur;
    for (long long it = 0;; ++it) {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(p) : "memory");
        if (cur >= v) return;
        __nanosleep(128);
        if (it > (1ll << 24)) {
            dbg[0] = 1u;
            dbg[1] = code;
            dbg[2] = R;
            dbg[3] = hh;
            dbg[4] = blockIdx.x;
            dbg[5] = cur;
            dbg[6] = v;
            __threadfence_system();
            asm volatile("trap;");
        }
    }
}
__global__ void __launch_bounds__(256) gram_jacobi_kernel(GramJacArgs a) {
    extern __shared__ double gsm[];
    double(*G)[kGPitch] = reinterpret_cast<double(*)[kGPitch]>(gsm);
    double(*J)[kGPitch] = reinterpret_cast<double(*)[kGPitch]>(gsm + kGP * kGPitch);
    double(*Cb)[kGCP] = reinterpret_cast<double(*)[kGCP]>(gsm + 2 * kGP * kGPitch);
    double(*Jb)[kGJP] = reinterpret_cast<double(*)[kGJP]>(gsm + 2 * kGP * kGPitch + kGP * kGCP);
    __shared__ double rcs[kGB], rsn[kGB];
    __shared__ int ract[kGB];
    __shared__ int s_any, s_rot;
    const int t = threadIdx.x;
    const int m = a.m, n = a.n, nb = a.nb;
    const double eps = 1e-15;
    volatile int* flags = a.flags;
    int sweep = 0;
    for (;;) {
        if (sweep >= kOneSidedSweepCap) {
            if (blockIdx.x == 0 && t == 0) flags[3] = RLRA_ECONV;
            break;
        }
        if (blockIdx.x == 0 && t == 0) flags[(sweep + 1) % 3] = 0;
        for (int r = 0; r < nb - 1; ++r) {
            for (int g = blockIdx.x; g < nb / 2; g += gridDim.x) {
                const int b1 = rr_col(g, r, nb), b2 = rr_col(nb - 1 - g, r, nb);
                const int bI = min(b1, b2), bJ = max(b1, b2);
                auto gcol = [&](int c) { return c < kGB ? bI * kGB + c : bJ * kGB + (c - kGB); };
                // ---- 1. Gram of the 64 columns on DMMA ----------------------
                // warp (wi, wj) owns G[wi*16 .. +16][wj*32 .. +32]
                const int warp = t >> 5, lane = t & 31, lr = lane >> 2, lc = lane & 3;
                const int wi = warp & 3, wj = warp >> 2;
                double acc[2][4][2];
#pragma unroll
                for (int f = 0; f < 2; ++f)
#pragma unroll
                    for (int g2 = 0; g2 < 4; ++g2) acc[f][g2][0] = acc[f][g2][1] = 0.0;
                double pre[8];
                auto load_chunk = [&](int k0) {
#pragma unroll
                    for (int it = 0; it < 8; ++it) {
                        const int e = t + it * 256, c = e >> 5, k = e & 31;
                        const int gc = gcol(c);
                        pre[it] = (gc < n && k0 + k < m) ? a.W[(k0 + k) + int64_t(gc) * a.ldw] : 0.0;
                    }
                };
                load_chunk(0);
                for (int k0 = 0; k0 < m; k0 += kGChunk) {
                    __syncthreads();
#pragma unroll
                    for (int it = 0; it < 8; ++it) {
                        const int e = t + it * 256;
                        Cb[e >> 5][e & 31] = pre[it];
                    }
                    __syncthreads();
                    if (k0 + kGChunk < m) load_chunk(k0 + kGChunk);
#pragma unroll
                    for (int kk = 0; kk < kGChunk; kk += 4) {
                        double af[2], bf[4];
#pragma unroll
                        for (int f = 0; f < 2; ++f) af[f] = Cb[wi * 16 + f * 8 + lr][kk + lc];
#pragma unroll
                        for (int g2 = 0; g2 < 4; ++g2) bf[g2] = Cb[wj * 32 + g2 * 8 + lr][kk + lc];
#pragma unroll
                        for (int f = 0; f < 2; ++f)
#pragma unroll
                            for (int g2 = 0; g2 < 4; ++g2) jac_dmma(acc[f][g2][0], acc[f][g2][1], af[f], bf[g2]);
                    }
                }
                __syncthreads();
#pragma unroll
                for (int f = 0; f < 2; ++f)
#pragma unroll
                    for (int g2 = 0; g2 < 4; ++g2)
#pragma unroll
                        for (int h = 0; h < 2; ++h) G[wi * 16 + f * 8 + lr][wj * 32 + g2 * 8 + 2 * lc + h] = acc[f][g2][h];
                for (int e = t; e < kGP * kGP; e += 256) J[e / kGP][e % kGP] = (e / kGP == e % kGP) ? 1.0 : 0.0;
                if (t == 0) s_rot = 0;
                __syncthreads();
                // ---- 2. inner Jacobi sweeps on G, accumulating J -------------
                for (int isw = 0; isw < a.inner_cap; ++isw) {
                    if (t == 0) s_any = 0;
                    __syncthreads();
                    for (int ir = 0; ir < kGP - 1; ++ir) {
                        if (t < kGB) {
                            const int c1 = rr_col(t, ir, kGP), c2 = rr_col(kGP - 1 - t, ir, kGP);
                            const int p = min(c1, c2), q = max(c1, c2);
                            int act = 0;
                            double c = 1.0, sn = 0.0;
                            if (gcol(q) < n && gcol(p) < n) {
                                const double app = G[p][p], aqq = G[q][q], apq = G[p][q];
                                if (app != 0.0 && aqq != 0.0 && fabs(apq) > eps * sqrt(app * aqq)) {
                                    const double zeta = (aqq - app) / (2.0 * apq);
                                    const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                                    c = 1.0 / sqrt(1.0 + tt * tt);
                                    sn = tt * c;
                                    act = 1;
                                    s_any = 1;
                                }
                            }
                            rcs[t] = c;
                            rsn[t] = sn;
                            ract[t] = act;
                        }
                        __syncthreads();
                        // columns of G and J
                        for (int e = t; e < kGB * kGP; e += 256) {
                            const int pi = e / kGP, i = e % kGP;
                            if (!ract[pi]) continue;
                            const int c1 = rr_col(pi, ir, kGP), c2 = rr_col(kGP - 1 - pi, ir, kGP);
                            const int p = min(c1, c2), q = max(c1, c2);
                            const double c = rcs[pi], sn = rsn[pi];
                            const double gp = G[i][p], gq = G[i][q];
                            G[i][p] = c * gp - sn * gq;
                            G[i][q] = sn * gp + c * gq;
                            const double jp = J[i][p], jq = J[i][q];
                            J[i][p] = c * jp - sn * jq;
                            J[i][q] = sn * jp + c * jq;
                        }
                        __syncthreads();
                        // rows of G
                        for (int e = t; e < kGB * kGP; e += 256) {
                            const int pi = e / kGP, i = e % kGP;
                            if (!ract[pi]) continue;
                            const int c1 = rr_col(pi, ir, kGP), c2 = rr_col(kGP - 1 - pi, ir, kGP);
                            const int p = min(c1, c2), q = max(c1, c2);
                            const double c = rcs[pi], sn = rsn[pi];
                            const double gp = G[p][i], gq = G[q][i];
                            G[p][i] = c * gp - sn * gq;
                            G[q][i] = sn * gp + c * gq;
                        }
                        __syncthreads();
                    }
                    if (!s_any) break;
                    if (t == 0) s_rot = 1;
                }
                __syncthreads();
                if (!s_rot) continue;  // uniform across the CTA
                if (t == 0) flags[sweep % 3] = 1;
                // ---- 3. W_p <- W_p J, V_p <- V_p J on DMMA (row chunks) -------
                for (int e = t; e < kGP * kGP; e += 256) Jb[e / kGP][e % kGP] = J[e / kGP][e % kGP];
                // warp (wr, wc) owns out[wr*16 .. +16][wc*16 .. +16] of a 32 x 64 chunk
                const int wr = warp & 1, wc = warp >> 1;
                for (int mat = 0; mat < 2; ++mat) {
                    double* X = mat == 0 ? a.W : a.V;
                    const int64_t ldx = mat == 0 ? a.ldw : a.ldv;
                    const int rows = mat == 0 ? m : n;
                    auto load_x = [&](int k0) {
#pragma unroll
                        for (int it = 0; it < 8; ++it) {
                            const int e = t + it * 256, c = e >> 5, k = e & 31, gc = gcol(c);
                            pre[it] = (gc < n && k0 + k < rows) ? X[(k0 + k) + int64_t(gc) * ldx] : 0.0;
                        }
                    };
                    load_x(0);
                    for (int k0 = 0; k0 < rows; k0 += kGChunk) {
                        __syncthreads();
#pragma unroll
                        for (int it = 0; it < 8; ++it) {
                            const int e = t + it * 256;
                            Cb[e >> 5][e & 31] = pre[it];
                        }
                        __syncthreads();
                        // the next chunk's rows are disjoint from this chunk's outputs
                        if (k0 + kGChunk < rows) load_x(k0 + kGChunk);
                        double o[2][2][2];
#pragma unroll
                        for (int f = 0; f < 2; ++f)
#pragma unroll
                            for (int g2 = 0; g2 < 2; ++g2) o[f][g2][0] = o[f][g2][1] = 0.0;
#pragma unroll
                        for (int kk = 0; kk < kGP; kk += 4) {
                            double af[2], bf[2];
#pragma unroll
                            for (int f = 0; f < 2; ++f) af[f] = Cb[kk + lc][wr * 16 + f * 8 + lr];
#pragma unroll
                            for (int g2 = 0; g2 < 2; ++g2) bf[g2] = Jb[kk + lc][wc * 16 + g2 * 8 + lr];
#pragma unroll
                            for (int f = 0; f < 2; ++f)
#pragma unroll
                                for (int g2 = 0; g2 < 2; ++g2) jac_dmma(o[f][g2][0], o[f][g2][1], af[f], bf[g2]);
                        }
#pragma unroll
                        for (int f = 0; f < 2; ++f) {
                            const int k = k0 + wr * 16 + f * 8 + lr;
#pragma unroll
                            for (int g2 = 0; g2 < 2; ++g2)
#pragma unroll
                                for (int h = 0; h < 2; ++h) {
                                    const int gj = gcol(wc * 16 + g2 * 8 + 2 * lc + h);
                                    if (gj < n && k < rows) X[k + int64_t(gj) * ldx] = o[f][g2][h];
                                }
                        }
                    }
                }
                __syncthreads();
            }
            grid_sync(a.bar);
        }
        const int rotated = flags[sweep % 3];
        ++sweep;
        if (!rotated || n < 2) break;
    }
    if (blockIdx.x == 0 && t == 0) flags[4] = sweep;
}

// ------------------------ Gram block Jacobi, shared-memory-resident pairs ---
// For l x l inputs with l up to ~1400 (the R-hat of rsvd_v2 at C1/C4/C5).
// Columns in blocks of BW; a sweep is nb-1 "cross" rounds (block pairs from a
// round-robin tournament; inside a visit BW steps rotate every (I_k, J_k+s)
// column pair) plus one "intra" round (blocks 2g, 2g+1; BW-1 tournament
// steps over the pairs inside each block), so every column pair is rotated
// exactly once per sweep — a cyclic ordering, as the reference's
// (core/jacobi.hpp:164-199), with its rotation formula, skip rule and
// "sweep without rotations" stop.  Per visit one CTA
//   1. stages the 2*BW columns in shared memory once and forms
//      G = W_p^T W_p on DMMA (each warp a row slice, upper 8x8 tiles; a
//      tile's two operand fragments are the same column-block loads);
//   2. runs the visit's steps on G: thread (k, l) owns the 2x2 block of
//      pairs (k, l), computes both pairs' rotations itself from the diagonal
//      entries (no serial parameter phase), updates its G block into the
//      other buffer and its J block in place — one barrier per step;
//   3. W_p J on DMMA straight from shared memory to W, and V_p <- V_p J.
// The one-sided variant (block_jacobi_kernel) re-reads all staged columns
// in every inner round and is shared-memory-bandwidth bound.
template <int BW>
struct BGram {
    static constexpr int C2 = 2 * BW;       // columns per pair
    static constexpr int NB8 = C2 / 8;      // 8-column blocks
    static constexpr int NT = NB8 * (NB8 + 1) / 2;  // upper 8x8 Gram tiles
    static constexpr int GP = C2 + 1;       // G / J pitch
    static constexpr int JP = C2 + 4;       // J pitch for the DMMA B fragments
    static constexpr int KF = C2 / 4;       // k-fragments of the apply
};

__host__ __device__ inline int bgram_rows(int m) { return (m + 31) & ~31; }    // 8 warps x k-steps of 4
__host__ __device__ inline int bgram_pitch(int m) { return bgram_rows(m) + 4; }  // == 4 mod 16: conflict-free

template <int BW>
size_t bgram_smem(int m) {
    using B = BGram<BW>;
    return sizeof(double) * (size_t(B::C2) * bgram_pitch(m) + 3 * B::C2 * B::GP + B::C2 * B::JP + 8 * B::NT * 64);
}

// 1/x and 1/sqrt(x) from the MUFU approximations (MUFU.RCP64H / RSQ64H, no
// special-case subroutine) plus three Newton steps: ~1 ulp on normal inputs
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    double e = fma(-hx * y, y, 0.5);
    y = fma(y, e, y);
    e = fma(-hx * y, y, 0.5);
    y = fma(y, e, y);
    const double r = fma(-x, y * y, 1.0);  // last step on the full residual
    return fma(0.5 * y, r, y);
}

// two Newton steps: ~1e-14 relative — for quantities whose rounding does not
// reach the rotation's orthogonality (hypot and 1/x inside t; c and s are
// formed from t consistently, c with the full-precision rsqrt_nr)
__device__ __forceinline__ double rcp_nr2(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ double rsqrt_nr2(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    double e = fma(-hx * y, y, 0.5);
    y = fma(y, e, y);
    e = fma(-hx * y, y, 0.5);
    return fma(y, e, y);
}

// OR-reduction barrier over the first `nthreads` threads (named barrier 1)
__device__ __forceinline__ int bar_or_partial(int nthreads, int pred) {
    int r;
    asm volatile(
        "{\n.reg .pred p, q;\nsetp.ne.s32 p, %1, 0;\nbar.red.or.pred q, 1, %2, p;\nselp.s32 %0, 1, 0, q;\n}\n"
        : "=r"(r)
        : "r"(pred), "r"(nthreads)
        : "memory");
    return r;
}

// The reference rotation (core/jacobi.hpp:170-180) for the pair with Gram
// entries (app, aqq, apq): skip unless |apq| > eps sqrt(app aqq); then
// t = sgn(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (aqq - app) / (2 apq),
// c = 1 / sqrt(1 + t^2), s = t c.
// Fast form, branch-free (the inner step is one dependent chain, so two of
// them interleave): t = |e| / (|d| + hypot(d, e)) with d = aqq - app,
// e = 2 apq — the same t — and the skip test on squares.  Returns false when
// a product is near over/underflow; the caller then takes jac_rotation_ref.
// An exactly orthogonal pair (apq == 0: every pair with a zero or padded
// column) is a plain skip on the fast path, as in the reference.
__device__ __forceinline__ bool jac_rotation_fast(double app, double aqq, double apq, double& c, double& s,
                                                  int& act) {
    const double pr = app * aqq, d = aqq - app, e = 2.0 * apq;
    const double h2 = fma(d, d, e * e);
    const bool ok = (pr > 1e-290 && pr < 1e290 && h2 > 1e-290 && h2 < 1e290) || apq == 0.0;
    act = apq * apq > 1e-30 * pr;
    const double h = h2 * rsqrt_nr2(h2);
    const double tm = fabs(e) * rcp_nr2(fabs(d) + h);
    const double t = (d == 0.0 || ((d > 0.0) == (e > 0.0))) ? tm : -tm;
    const double cc = rsqrt_nr(fma(t, t, 1.0));
    c = act ? cc : 1.0;
    s = act ? t * cc : 0.0;
    return ok;
}
struct RotRef {
    double c, s;
    int act;
};
// (returned by value: the call leaves the caller's rotation in registers)
__device__ __noinline__ RotRef jac_rotation_ref_v(double app, double aqq, double apq) {
    RotRef r{1.0, 0.0, 0};
    if (!(app != 0.0 && aqq != 0.0 && fabs(apq) > 1e-15 * sqrt(app * aqq))) return r;
    const double zeta = (aqq - app) / (2.0 * apq);
    const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
    r.c = 1.0 / sqrt(1.0 + t * t);
    r.s = t * r.c;
    r.act = 1;
    return r;
}
__device__ __forceinline__ int jac_rotation_ref(double app, double aqq, double apq, double& c, double& s) {
    const RotRef r = jac_rotation_ref_v(app, aqq, apq);
    c = r.c;
    s = r.s;
    return r.act;
}

// pair k of step st in a cross (I_k, J_{k+st}) or intra (tournament inside
// each block) visit; returns p | q << 8, p < q
template <int BW>
__device__ __forceinline__ int bgram_pair(bool intra, int k, int st) {
    if (!intra) return k | ((BW + (k + st) % BW) << 8);
    const int half = k / (BW / 2), kk = k % (BW / 2), base = half * BW;
    const int c1 = base + rr_col(kk, st, BW), c2 = base + rr_col(BW - 1 - kk, st, BW);
    return min(c1, c2) | (max(c1, c2) << 8);
}

// Stage the 2*BW columns (global pitch ld, even; rows2 = rows rounded to 2)
// of blocks bI, bJ into Xs (pitch P, Mp rows): thread 0 waits until both
// blocks reached version `need` (their last writers published), then issues
// one bulk copy per column; rows >= rows2 and padded columns are zeroed.
template <int BW>
__device__ __forceinline__ void bgram_stage(double* Xs, int P, int Mp, const double* X, int64_t ld, int rows2,
                                            int n, int bI, int bJ, const unsigned* ver, unsigned need,
                                            uint64_t* bar, unsigned& phase) {
    constexpr int C2 = 2 * BW;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    auto gcol = [&](int c) { return c < BW ? bI * BW + c : bJ * BW + (c - BW); };
    if (t == 0) {
        jb_wait_at_least(ver + bI, need);
        jb_wait_at_least(ver + bJ, need);
        // acquire (this SM's L1 invalidated); the writers' generic stores and
        // this CTA's generic smem reads of the last visit ordered before the
        // async-proxy copies
        asm volatile("fence.acq_rel.gpu;\nfence.proxy.async.global;\nfence.proxy.async.shared::cta;\n" ::: "memory");
        const int nv = max(0, min(BW, n - bI * BW)) + max(0, min(BW, n - bJ * BW));
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(jb_smem(bar)),
                     "r"(unsigned(nv) * unsigned(rows2) * 8u)
                     : "memory");
        for (int c = 0; c < C2; ++c) {
            const int gc = gcol(c);
            if (gc < n) jb_bulk_load(Xs + size_t(c) * P, X + int64_t(gc) * ld, unsigned(rows2) * 8u, bar);
        }
    }
    for (int c = warp; c < C2; c += 8) {
        double* dst = Xs + size_t(c) * P;
        for (int i = (gcol(c) < n ? rows2 : 0) + lane; i < Mp; i += 32) dst[i] = 0.0;
    }
    jb_mbar_wait(bar, phase);
    phase ^= 1u;
    __syncthreads();
}

// X(rows, cols of the pair) <- Xs * J on DMMA (Xs staged, Jb pitch JP),
// written straight to global; warps take pairs of 8-row slabs
template <int BW>
__device__ __forceinline__ void bgram_apply(const double* Xs, int P, int Mp, const double* Jb, double* X, int64_t ld,
                                            int rows, int n, int bI, int bJ) {
    using B = BGram<BW>;
    constexpr int NB8 = B::NB8, JP = B::JP, KF = B::KF;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
    auto gcol = [&](int c) { return c < BW ? bI * BW + c : bJ * BW + (c - BW); };
    double bf[KF][NB8];
#pragma unroll
    for (int kf = 0; kf < KF; ++kf)
#pragma unroll
        for (int ct = 0; ct < NB8; ++ct) bf[kf][ct] = Jb[(4 * kf + lc) * JP + ct * 8 + lr];
    int ocol[NB8][2];
#pragma unroll
    for (int ct = 0; ct < NB8; ++ct)
#pragma unroll
        for (int h = 0; h < 2; ++h) ocol[ct][h] = gcol(ct * 8 + 2 * lc + h);
    for (int sl0 = 2 * warp; sl0 < Mp / 8; sl0 += 16) {  // Mp / 8 is a multiple of 4
        double af[2][KF];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int kf = 0; kf < KF; ++kf) af[u][kf] = Xs[(4 * kf + lc) * P + (sl0 + u) * 8 + lr];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int row = (sl0 + u) * 8 + lr;
#pragma unroll
            for (int ct = 0; ct < NB8; ++ct) {
                double o0 = 0.0, o1 = 0.0;
#pragma unroll
                for (int kf = 0; kf < KF; ++kf) jac_dmma(o0, o1, af[u][kf], bf[kf][ct]);
                if (row < rows) {
                    if (ocol[ct][0] < n) X[row + int64_t(ocol[ct][0]) * ld] = o0;
                    if (ocol[ct][1] < n) X[row + int64_t(ocol[ct][1]) * ld] = o1;
                }
            }
        }
    }
}

__device__ __forceinline__ void jb_publish(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// a relaxed store for a publish that follows a gpu-scope fence of the same
// thread (the fence already orders every earlier write and every write it
// observed before it)
__device__ __forceinline__ void jb_store_relaxed(unsigned* p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Gram G0 = Xs^T Xs of a staged pair (C2 columns, pitch P, Mp rows) on DMMA:
// warp w sums rows [w*Mp/8, (w+1)*Mp/8) for the upper 8x8 tiles (a tile's two
// operand fragments are the same column-block loads), the 8 partials (Pb)
// summed in a fixed order, G0 mirrored; J <- I.  The caller synchronises.
template <int BW>
__device__ __forceinline__ void bgram_gram(const double* Ws, int P, int Mp, double* Pb, double* G0, double* J) {
    using B = BGram<BW>;
    constexpr int C2 = B::C2, NB8 = B::NB8, NT = B::NT, GP = B::GP;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31, lr = lane >> 2, lc = lane & 3;
    {
        // two accumulator sets (even / odd k-steps) halve the DMMA chain
        double acc[2][NT][2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int u = 0; u < NT; ++u) acc[h][u][0] = acc[h][u][1] = 0.0;
        const int k1 = (warp + 1) * (Mp / 8);
        for (int k = warp * (Mp / 8); k < k1; k += 8) {  // Mp / 8 is a multiple of 4
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (h == 1 && k + 4 >= k1) break;
                double f[NB8];
#pragma unroll
                for (int bb = 0; bb < NB8; ++bb) f[bb] = Ws[(bb * 8 + lr) * P + k + 4 * h + lc];
                int u = 0;
#pragma unroll
                for (int bi = 0; bi < NB8; ++bi)
#pragma unroll
                    for (int bj = bi; bj < NB8; ++bj, ++u) jac_dmma(acc[h][u][0], acc[h][u][1], f[bi], f[bj]);
            }
        }
#pragma unroll
        for (int u = 0; u < NT; ++u) {
            Pb[(warp * NT + u) * 64 + lr * 8 + 2 * lc] = acc[0][u][0] + acc[1][u][0];
            Pb[(warp * NT + u) * 64 + lr * 8 + 2 * lc + 1] = acc[0][u][1] + acc[1][u][1];
        }
    }
    __syncthreads();
    for (int e = t; e < NT * 64; e += blockDim.x) {
        const int u = e >> 6, w = e & 63;
        int bi = 0, rem = u;
        while (rem >= NB8 - bi) rem -= NB8 - bi++;
        const int bj = bi + rem;
        double sum = 0.0;
#pragma unroll
        for (int ww = 0; ww < 8; ++ww) sum += Pb[(ww * NT + u) * 64 + w];
        const int row = bi * 8 + (w >> 3), col = bj * 8 + (w & 7);
        G0[row * GP + col] = sum;
        G0[col * GP + row] = sum;
    }
    for (int e = t; e < C2 * C2; e += blockDim.x) J[(e / C2) * GP + e % C2] = (e / C2 == e % C2) ? 1.0 : 0.0;
}

// The visit's steps on G (double-buffered G0) accumulating J, by the BW*BW
// threads t < BW*BW: thread (k, l) owns the 2x2 block of pairs (k, l),
// computes both pairs' rotations itself from the diagonal entries (no serial
// parameter phase), updates its G block into the other buffer and its J block
// in place — one barrier (named barrier 1 unless BW*BW == 256) per step.
// Returns whether any pair rotated (the same value on every caller thread).
template <int BW, bool INTRA>
__device__ __forceinline__ int bgram_steps_t(double* G0, double* J) {
    constexpr bool intra = INTRA;
    using B = BGram<BW>;
    constexpr int C2 = B::C2, GP = B::GP;
    const int t = threadIdx.x;
    int rot = 0;
    const int k = t / BW, l = t % BW;
    constexpr int nsteps = INTRA ? BW - 1 : BW;
#pragma unroll
    for (int st = 0; st < nsteps; ++st) {
        const double* Gc = G0 + (st & 1) * C2 * GP;
        double* Gn = G0 + ((st & 1) ^ 1) * C2 * GP;
        int act = 0;
        {
            const int pqk = bgram_pair<BW>(intra, k, st), pql = bgram_pair<BW>(intra, l, st);
            const int pk = pqk & 255, qk = pqk >> 8, pl = pql & 255, ql = pql >> 8;
            // (a padded column's Gram entries are 0: never rotated)
            const double kpp = Gc[pk * GP + pk], kqq = Gc[qk * GP + qk], kpq = Gc[pk * GP + qk];
            const double lpp = Gc[pl * GP + pl], lqq = Gc[ql * GP + ql], lpq = Gc[pl * GP + ql];
            // this thread's J and G blocks: loaded under the rotation chain
            // (independent of it), updated without branches (a skipped
            // rotation keeps the values: selects, not arithmetic)
            const double j0 = J[pk * GP + pl], j1 = J[pk * GP + ql];
            const double j2 = J[qk * GP + pl], j3 = J[qk * GP + ql];
            double b00 = Gc[pk * GP + pl], b01 = Gc[pk * GP + ql];
            double b10 = Gc[qk * GP + pl], b11 = Gc[qk * GP + ql];
            double ck, sk, cl, sl;
            int ak, al;
            const bool okk = jac_rotation_fast(kpp, kqq, kpq, ck, sk, ak);
            const bool okl = jac_rotation_fast(lpp, lqq, lpq, cl, sl, al);
            if (!okk) ak = jac_rotation_ref(kpp, kqq, kpq, ck, sk);
            if (!okl) al = jac_rotation_ref(lpp, lqq, lpq, cl, sl);
            act = (k == l) ? ak : 0;
            rot |= act;
            if (al) {  // J <- J R_l on rows {pk, qk}
                J[pk * GP + pl] = cl * j0 - sl * j1;
                J[pk * GP + ql] = sl * j0 + cl * j1;
                J[qk * GP + pl] = cl * j2 - sl * j3;
                J[qk * GP + ql] = sl * j2 + cl * j3;
            }
            {
                const double x0 = cl * b00 - sl * b01, x1 = sl * b00 + cl * b01;
                const double x2 = cl * b10 - sl * b11, x3 = sl * b10 + cl * b11;
                b00 = al ? x0 : b00, b01 = al ? x1 : b01, b10 = al ? x2 : b10, b11 = al ? x3 : b11;
                const double y0 = ck * b00 - sk * b10, y2 = sk * b00 + ck * b10;
                const double y1 = ck * b01 - sk * b11, y3 = sk * b01 + ck * b11;
                b00 = ak ? y0 : b00, b01 = ak ? y1 : b01, b10 = ak ? y2 : b10, b11 = ak ? y3 : b11;
            }
            if (k <= l) {  // G block (k, l) <- R_k^T B R_l, mirrored
                Gn[pk * GP + pl] = b00;
                Gn[pk * GP + ql] = b01;
                Gn[qk * GP + pl] = b10;
                Gn[qk * GP + ql] = b11;
                Gn[pl * GP + pk] = b00;
                Gn[ql * GP + pk] = b01;
                Gn[pl * GP + qk] = b10;
                Gn[ql * GP + qk] = b11;
            }
        }
        // plain barrier per step; the rotation flags are OR-reduced once below
        if (BW * BW == 256)
            __syncthreads();
        else
            asm volatile("bar.sync 1, %0;\n" ::"n"(BW * BW) : "memory");
    }
    return (BW * BW == 256) ? __syncthreads_or(rot) : bar_or_partial(BW * BW, rot);
}
template <int BW>
__device__ __forceinline__ int bgram_steps(double* G0, double* J, bool intra) {
    return intra ? bgram_steps_t<BW, true>(G0, J) : bgram_steps_t<BW, false>(G0, J);
}

// V(rows, cols of the pair) <- V * Jb on DMMA, read and written through L2
// (__ldcg: other CTAs wrote these columns in earlier rounds), by warps
// [w0, w0 + nw) with 8-row slabs in flight
template <int BW>
__device__ __forceinline__ void bgram_apply_l2(const double* Jb, double* V, int64_t ldv, int n, int bI, int bJ,
                                               int w0, int nw) {
    using B = BGram<BW>;
    constexpr int NB8 = B::NB8, JP = B::JP, KF = B::KF;
    const int warp = int(threadIdx.x >> 5) - w0, lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
    auto gcol = [&](int c) { return c < BW ? bI * BW + c : bJ * BW + (c - BW); };
    double bf[KF][NB8];
#pragma unroll
    for (int kf = 0; kf < KF; ++kf)
#pragma unroll
        for (int ct = 0; ct < NB8; ++ct) bf[kf][ct] = Jb[(4 * kf + lc) * JP + ct * 8 + lr];
    int icol[KF], ocol[NB8][2];
#pragma unroll
    for (int kf = 0; kf < KF; ++kf) icol[kf] = gcol(4 * kf + lc);
#pragma unroll
    for (int ct = 0; ct < NB8; ++ct)
#pragma unroll
        for (int h = 0; h < 2; ++h) ocol[ct][h] = gcol(ct * 8 + 2 * lc + h);
    constexpr int U = 32 / KF;  // V slabs (8 rows) in flight per warp
    for (int sl0 = warp * U; sl0 < (n + 7) / 8; sl0 += nw * U) {
        double af[U][KF];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int row = (sl0 + u) * 8 + lr;
#pragma unroll
            for (int kf = 0; kf < KF; ++kf)
                af[u][kf] = (row < n && icol[kf] < n) ? __ldcg(V + row + int64_t(icol[kf]) * ldv) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int row = (sl0 + u) * 8 + lr;
#pragma unroll
            for (int ct = 0; ct < NB8; ++ct) {
                double o0 = 0.0, o1 = 0.0;
#pragma unroll
                for (int kf = 0; kf < KF; ++kf) jac_dmma(o0, o1, af[u][kf], bf[kf][ct]);
                if (row < n) {
                    if (ocol[ct][0] < n) __stcg(V + row + int64_t(ocol[ct][0]) * ldv, o0);
                    if (ocol[ct][1] < n) __stcg(V + row + int64_t(ocol[ct][1]) * ldv, o1);
                }
            }
        }
    }
}

// a.helpers == 0: CTA g runs pair slots g, g + grid, ... and applies J to
// both W and V.  a.helpers == 1 (grid = nb): CTAs [0, nb/2) are the pair
// owners (W: stage, Gram, steps, publish J, W J) and CTAs [nb/2, nb) their
// V helpers (prefetch the pair's V columns while the owner works, then V J):
// V's L2 traffic leaves the owners' critical path and runs on another SM.
// Versions: ver[b] = rounds of block b's W columns done, ver[nb + b] = of
// its V columns (helpers; == ver[b] without helpers); jrdy[g] = 2 (R + 1) +
// rotated, jcon[g] = R + 1 once the helper copied round R's J (the owner
// reuses J slot R & 1 two rounds later).
template <int BW>
__global__ void __launch_bounds__(256, 1) bgram_jacobi_kernel(GramJacArgs a) {
    using B = BGram<BW>;
    constexpr int C2 = B::C2, NB8 = B::NB8, NT = B::NT, GP = B::GP, JP = B::JP;
    static_assert(BW * BW <= 256, "one thread per 2x2 pair block");
    extern __shared__ double bsm[];
    const int m = a.m, n = a.n, nb = a.nb, np = nb / 2;
    const int Mp = bgram_rows(m), P = bgram_pitch(m);
    double* Ws = bsm;                               // C2 columns, pitch P (helpers: V columns)
    double* G0 = Ws + size_t(C2) * P;               // C2 x GP, two buffers
    double* J = G0 + 2 * C2 * GP;                   // C2 x GP
    double* Jb = J + C2 * GP;                       // C2 x JP
    double* Pb = Jb + C2 * JP;                      // 8 warps x NT tiles x 64 partial Grams
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31, lr = lane >> 2, lc = lane & 3;
    const bool helpers = a.helpers != 0, helper = helpers && int(blockIdx.x) >= np;
    const int g0 = helper ? int(blockIdx.x) - np : int(blockIdx.x), gstep = helpers ? np : int(gridDim.x);
    unsigned* wver = a.ver;
    unsigned* vver = helpers ? a.ver + nb : a.ver;
    unsigned* jrdy = a.ver + 2 * nb;
    unsigned* jcon = jrdy + np;
    __shared__ __align__(8) uint64_t stage_bar;
    __shared__ int s_rot;
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(jb_smem(&stage_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    unsigned stage_phase = 0, R = 0;  // R: global round (the version every block reaches)
    volatile int* flags = a.flags;
    const bool clk = a.phase_clk != nullptr && blockIdx.x == 0 && t == 0;
    long long ph[6] = {0, 0, 0, 0, 0, 0}, c0 = clock64();
    auto mark = [&](int i) {
        if (clk) {
            const long long c1 = clock64();
            ph[i] += c1 - c0;
            c0 = c1;
        }
    };
    int sweep = 0;
    for (;;) {
        if (sweep >= kOneSidedSweepCap) {
            if (blockIdx.x == 0 && t == 0) flags[3] = RLRA_ECONV;
            break;
        }
        if (blockIdx.x == 0 && t == 0) flags[(sweep + 1) % 3] = 0;
        for (int r = 0; r < nb; ++r) {
            const bool intra = r == nb - 1;
            for (int g = g0; g < np; g += gstep) {
                int bI = 2 * g, bJ = 2 * g + 1;
                if (!intra) {
                    const int b1 = rr_col(g, r, nb), b2 = rr_col(nb - 1 - g, r, nb);
                    bI = min(b1, b2);
                    bJ = max(b1, b2);
                }
                auto gcol = [&](int c) { return c < BW ? bI * BW + c : bJ * BW + (c - BW); };
                if (helper) {
                    // ---- V helper: prefetch V_p, take the owner's J, V_p J ------
                    bgram_stage<BW>(Ws, P, bgram_rows(n), a.V, a.ldv, (n + 1) & ~1, n, bI, bJ, vver, R, &stage_bar,
                                    stage_phase);
                    if (t == 0) {
                        unsigned cur, ns = 32;
                        for (;;) {
                            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(jrdy + g) : "memory");
                            if (cur >= 2 * (R + 1)) break;
                            __nanosleep(ns);
                            ns = ns < 128 ? ns * 2 : 128;
                        }
                        asm volatile("fence.acq_rel.gpu;" ::: "memory");
                        s_rot = int(cur & 1u);
                    }
                    __syncthreads();
                    const int rot = s_rot;
                    if (rot) {
                        const double* js = a.jbuf + (size_t(g) * 2 + (R & 1)) * C2 * C2;
                        for (int e = t; e < C2 * C2; e += 256) Jb[(e / C2) * JP + e % C2] = __ldcg(js + e);
                    }
                    __syncthreads();
                    if (t == 0) jb_publish(jcon + g, R + 1);
                    if (rot) bgram_apply<BW>(Ws, P, bgram_rows(n), Jb, a.V, a.ldv, n, n, bI, bJ);
                    __syncthreads();
                    if (t == 0) {
                        __threadfence();
                        jb_publish(vver + bI, R + 1);
                        jb_publish(vver + bJ, R + 1);
                    }
                    continue;
                }
                // ---- owner: stage W_p -------------------------------------------
                bgram_stage<BW>(Ws, P, Mp, a.W, a.ldw, (m + 1) & ~1, n, bI, bJ, wver, R, &stage_bar, stage_phase);
                mark(0);
                // ---- 1. Gram: warp w sums rows [w*Mp/8, (w+1)*Mp/8) ------------
                bgram_gram<BW>(Ws, P, Mp, Pb, G0, J);
                __syncthreads();
                mark(1);
                // ---- 2. the visit's steps on G: thread (k, l) owns pair block (k, l)
                int rot = t < BW * BW ? bgram_steps<BW>(G0, J, intra) : 0;
                rot = __syncthreads_or(rot);
                mark(2);
                if (rot && t == 0) flags[sweep % 3] = 1;
                if (helpers) {
                    // hand J to the V helper (slot R & 1, free once round R - 2's J was taken)
                    double* js = a.jbuf + (size_t(g) * 2 + (R & 1)) * C2 * C2;
                    if (rot) {
                        if (t == 0) jb_wait_at_least(jcon + g, R >= 1 ? R - 1 : 0);
                        __syncthreads();
                        for (int e = t; e < C2 * C2; e += 256) __stcg(js + e, J[(e / C2) * GP + e % C2]);
                    }
                    __syncthreads();
                    if (t == 0) {
                        __threadfence();
                        jb_publish(jrdy + g, 2 * (R + 1) + (rot ? 1u : 0u));
                    }
                }
                if (rot) {  // uniform across the CTA
                    for (int e = t; e < C2 * C2; e += 256) Jb[(e / C2) * JP + e % C2] = J[(e / C2) * GP + e % C2];
                    __syncthreads();
                    // ---- 3. W_p <- W_p J (shared -> global); V_p <- V_p J here
                    // without helpers (V from L2, 8-row slabs in flight) ------------
                    bgram_apply<BW>(Ws, P, Mp, Jb, a.W, a.ldw, m, n, bI, bJ);
                    mark(3);
                    if (!helpers) {
                        constexpr int KF = B::KF;
                        double bf[KF][NB8];
#pragma unroll
                        for (int kf = 0; kf < KF; ++kf)
#pragma unroll
                            for (int ct = 0; ct < NB8; ++ct) bf[kf][ct] = Jb[(4 * kf + lc) * JP + ct * 8 + lr];
                        int icol[KF], ocol[NB8][2];
#pragma unroll
                        for (int kf = 0; kf < KF; ++kf) icol[kf] = gcol(4 * kf + lc);
#pragma unroll
                        for (int ct = 0; ct < NB8; ++ct)
#pragma unroll
                            for (int h = 0; h < 2; ++h) ocol[ct][h] = gcol(ct * 8 + 2 * lc + h);
                        constexpr int U = 32 / KF;  // V slabs (8 rows) in flight per warp
                        for (int sl0 = warp * U; sl0 < (n + 7) / 8; sl0 += 8 * U) {
                            double af[U][KF];
#pragma unroll
                            for (int u = 0; u < U; ++u) {
                                const int row = (sl0 + u) * 8 + lr;
#pragma unroll
                                for (int kf = 0; kf < KF; ++kf)
                                    af[u][kf] = (row < n && icol[kf] < n) ? a.V[row + int64_t(icol[kf]) * a.ldv] : 0.0;
                            }
#pragma unroll
                            for (int u = 0; u < U; ++u) {
                                const int row = (sl0 + u) * 8 + lr;
#pragma unroll
                                for (int ct = 0; ct < NB8; ++ct) {
                                    double o0 = 0.0, o1 = 0.0;
#pragma unroll
                                    for (int kf = 0; kf < KF; ++kf) jac_dmma(o0, o1, af[u][kf], bf[kf][ct]);
                                    if (row < n) {
                                        if (ocol[ct][0] < n) a.V[row + int64_t(ocol[ct][0]) * a.ldv] = o0;
                                        if (ocol[ct][1] < n) a.V[row + int64_t(ocol[ct][1]) * a.ldv] = o1;
                                    }
                                }
                            }
                        }
                    }
                }
                // publish: both blocks' W (and V without helpers) reached round R + 1
                __syncthreads();
                if (t == 0) {
                    __threadfence();
                    jb_publish(wver + bI, R + 1);
                    jb_publish(wver + bJ, R + 1);
                }
                mark(4);
            }
            ++R;
        }
        grid_sync(a.bar);  // once per sweep: every CTA sees the sweep's rotation flag
        mark(5);
        const int rotated = flags[sweep % 3];
        ++sweep;
        if (!rotated || n < 2) break;
    }
    if (blockIdx.x == 0 && t == 0) flags[4] = sweep;
    if (clk)
        for (int i = 0; i < 6; ++i) a.phase_clk[i] = ph[i];
}

// ------------------ cluster-resident Gram block Jacobi (l <= 256, one cluster) ---
// The bgram schedule (blocks of BW = 8 columns, nb - 1 cross rounds + one
// intra round per sweep, every column pair once per sweep, the same Gram /
// steps arithmetic and stop rule) with the np = nb / 2 <= 16 pair CTAs
// forming ONE thread-block cluster, so W never leaves shared memory.  Per
// round a CTA
//   1. waits for its pair's columns (an mbarrier completed by the senders'
//      st.async bytes) and forms G = W_p^T W_p (DMMA),
//   2. runs the steps on G (2 warps),
//   3. sends W_p J (or W_p unchanged) straight into the shared memory of the
//      CTAs owning each block next round (st.async, double-buffered), and logs
//      J (jlog, one slot per (sweep parity, round, pair); rlog = rotated).
// Cross-CTA ordering: the data's own mbarrier (RAW) and one split cluster
// barrier per round, relaxed, for buffer reuse (WAR); a release/acquire
// cluster barrier once per sweep carries the rotation flag (a word in CTA
// 0's shared memory) and publishes the sweep's log.  V is off the critical
// path: CTA g keeps V's rows [16 g, 16 g + 16) in shared memory (starting as
// I), and while 2 warps run round r's steps the other 6 replay round r of
// the PREVIOUS sweep's log on those rows (DMMA).  The last sweep rotates
// nothing, so V is complete when the loop stops.
struct CGramArgs {
    double* W;
    int64_t ldw;
    int m, n;
    int nb;                // column blocks (even, <= 32)
    double* V;             // n x n
    int64_t ldv;
    double* jlog;          // [2][nb][np] C2 x C2 J, row-major (k, c)
    unsigned char* rlog;   // [2][nb][np] rotated
    int* flags;            // [3] status, [4] sweeps used
    long long* phase_clk;  // optional: CTA 0's clock64 per phase (RLRA_JACOBI_PHASES)
};

constexpr int kCgVRows = 16, kCgVP = kCgVRows + 4;  // V rows per CTA; column pitch (== 4 mod 16)

template <int BW>
size_t cgram_smem(int m, int nb) {
    using B = BGram<BW>;
    return sizeof(double) * (size_t(2) * B::C2 * bgram_pitch(m) + 3 * B::C2 * B::GP + B::C2 * B::JP +
                             8 * B::NT * 64 + size_t(nb) * BW * kCgVP);
}

__device__ __forceinline__ unsigned cg_map(const void* p, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(jb_smem(p)), "r"(rank));
    return r;
}
// 16 bytes into a peer's shared memory, completing on the peer's mbarrier
__device__ __forceinline__ void cg_st_async(unsigned addr, double v0, double v1, unsigned bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(addr),
                 "d"(v0), "d"(v1), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void cg_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cg_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cg_arrive_release() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cg_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }

template <int BW>
__global__ void __launch_bounds__(256, 1) cgram_jacobi_kernel(CGramArgs a) {
    using B = BGram<BW>;
    constexpr int C2 = B::C2, NB8 = B::NB8, GP = B::GP, JP = B::JP, KF = B::KF;
    static_assert(BW == 8, "one 8-column tile per block half");
    extern __shared__ double csm[];
    const int m = a.m, n = a.n, nb = a.nb, np = nb / 2;
    const int Mp = bgram_rows(m), P = bgram_pitch(m);
    double* Wb0 = csm;                      // 2 buffers of C2 columns, pitch P
    double* G0 = Wb0 + size_t(2) * C2 * P;  // C2 x GP, two buffers
    double* J = G0 + 2 * C2 * GP;           // C2 x GP
    double* Jb = J + C2 * GP;               // C2 x JP (DMMA B operand)
    double* Pb = Jb + C2 * JP;              // 8 warps x NT tiles x 64 partial Grams
    double* Vs = Pb + 8 * B::NT * 64;       // V rows [16 g, 16 g + 16), column-major, pitch kCgVP
    __shared__ unsigned char own[32 * 32];  // own[r * nb + b] = owner CTA << 1 | slot
    __shared__ unsigned char prs[32 * 16 * 2];  // [r][pair] -> bI, bJ
    __shared__ __align__(8) uint64_t inbar[2];
    __shared__ unsigned sflag[2];  // CTA 0: rotated-in-sweep (sweep parity)
    __shared__ int s_stop;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31, lr = lane >> 2, lc = lane & 3;
    const int g = int(blockIdx.x);
    const unsigned in_bytes = unsigned(C2) * unsigned(Mp) * 8u;
    auto pair_of = [&](int gg, int r, int& bI, int& bJ) {
        if (r == nb - 1) {
            bI = 2 * gg;
            bJ = 2 * gg + 1;
        } else {
            const int b1 = rr_col(gg, r, nb), b2 = rr_col(nb - 1 - gg, r, nb);
            bI = min(b1, b2);
            bJ = max(b1, b2);
        }
    };
    for (int e = t; e < np * nb; e += blockDim.x) {
        const int r = e / np, gg = e % np;
        int bI, bJ;
        pair_of(gg, r, bI, bJ);
        own[r * nb + bI] = (unsigned char)(gg << 1);
        own[r * nb + bJ] = (unsigned char)(gg << 1 | 1);
        prs[2 * (r * np + gg)] = (unsigned char)bI;
        prs[2 * (r * np + gg) + 1] = (unsigned char)bJ;
    }
    const int vr0 = g * kCgVRows;
    for (int e = t; e < nb * BW * kCgVP; e += blockDim.x) {
        const int c = e / kCgVP, i = e % kCgVP;
        Vs[e] = (i < kCgVRows && vr0 + i == c) ? 1.0 : 0.0;
    }
    if (t == 0) {
        sflag[0] = sflag[1] = 0u;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(jb_smem(&inbar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(jb_smem(&inbar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // round 0's pair from global W (rows >= m and padded columns zero)
    {
        int bI, bJ;
        pair_of(g, 0, bI, bJ);
        for (int e = t; e < C2 * Mp; e += blockDim.x) {
            const int c = e / Mp, i = e % Mp;
            const int gc = c < BW ? bI * BW + c : bJ * BW + (c - BW);
            Wb0[size_t(c) * P + i] = (gc < n && i < m) ? a.W[i + int64_t(gc) * a.ldw] : 0.0;
        }
    }
    __syncthreads();
    cg_sync();
    cg_arrive_relaxed();  // pairs with round 0's wait
    int sweep = 0, R = 0;
    bool econv = false;
    const bool clk = a.phase_clk != nullptr && g == 0 && t == 0;
    long long ph[7] = {0, 0, 0, 0, 0, 0, 0}, c0 = clock64();
    auto mark = [&](int i) {
        if (clk) {
            const long long c1 = clock64();
            ph[i] += c1 - c0;
            c0 = c1;
        }
    };
    for (;;) {
        if (sweep >= kOneSidedSweepCap) {
            econv = true;
            break;
        }
        for (int r = 0; r < nb; ++r, ++R) {
            const bool intra = r == nb - 1;
            int bI, bJ;
            pair_of(g, r, bI, bJ);
            double* Ws = Wb0 + size_t(R & 1) * C2 * P;
            double* Wn = Wb0 + size_t((R & 1) ^ 1) * C2 * P;
            // this round's columns (sent last round), then announce next round's
            if (t == 0) {
                if (R > 0) jb_mbar_wait(&inbar[R & 1], unsigned((R - 1) >> 1) & 1u);
                asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                                 jb_smem(&inbar[(R & 1) ^ 1])),
                             "r"(in_bytes)
                             : "memory");
            }
            __syncthreads();
            mark(0);
            // ---- 1. Gram of the resident pair --------------------------------
            bgram_gram<BW>(Ws, P, Mp, Pb, G0, J);
            __syncthreads();
            mark(1);
            // ---- 2. steps (the BW * BW pair-block owners) || V replay ---------
            int rot = 0;
            if (t < BW * BW) {
                rot = bgram_steps<BW>(G0, J, intra);
            } else if (sweep > 0) {
                // round r of the previous sweep's log on this CTA's V rows:
                // task = (8-row tile rt, pair gg), pairs own disjoint columns
                const size_t base = (size_t((sweep - 1) & 1) * nb + r) * np;
                for (int task = warp - (BW * BW) / 32; task < 2 * np; task += 8 - (BW * BW) / 32) {
                    const int rt = task & 1, gg = task >> 1;
                    if (!__ldcg(a.rlog + base + gg)) continue;
                    const int cI = prs[2 * (r * np + gg)] * BW, cJ = prs[2 * (r * np + gg) + 1] * BW;
                    const double* Jg = a.jlog + (base + gg) * C2 * C2;
                    double af[KF], bf[KF][NB8];
#pragma unroll
                    for (int kf = 0; kf < KF; ++kf) {
                        const int k = 4 * kf + lc;
                        af[kf] = Vs[(k < BW ? cI + k : cJ + k - BW) * kCgVP + rt * 8 + lr];
#pragma unroll
                        for (int ct = 0; ct < NB8; ++ct) bf[kf][ct] = __ldcg(Jg + k * C2 + ct * 8 + lr);
                    }
#pragma unroll
                    for (int ct = 0; ct < NB8; ++ct) {
                        double o0 = 0.0, o1 = 0.0;
#pragma unroll
                        for (int kf = 0; kf < KF; ++kf) jac_dmma(o0, o1, af[kf], bf[kf][ct]);
                        const int c = (ct == 0 ? cI : cJ) + 2 * lc;
                        Vs[c * kCgVP + rt * 8 + lr] = o0;
                        Vs[(c + 1) * kCgVP + rt * 8 + lr] = o1;
                    }
                }
            }
            rot = __syncthreads_or(rot);
            mark(2);
            // ---- 3. W_p J (or W_p) into the next owners' buffers; log J ------
            const int rn = r + 1 == nb ? 0 : r + 1;
            const unsigned oI = own[rn * nb + bI], oJ = own[rn * nb + bJ];
            const unsigned dst[2] = {cg_map(Wn + size_t(oI & 1u) * BW * P, oI >> 1),
                                     cg_map(Wn + size_t(oJ & 1u) * BW * P, oJ >> 1)};
            const unsigned dbar[2] = {cg_map(&inbar[(R & 1) ^ 1], oI >> 1), cg_map(&inbar[(R & 1) ^ 1], oJ >> 1)};
            const size_t slot = (size_t(sweep & 1) * nb + r) * np + g;
            if (t == 0) a.rlog[slot] = rot ? 1 : 0;
            if (rot) {
                for (int e = t; e < C2 * C2; e += blockDim.x) {
                    const double v = J[(e / C2) * GP + e % C2];
                    Jb[(e / C2) * JP + e % C2] = v;
                    a.jlog[slot * C2 * C2 + e] = v;
                }
                __syncthreads();
            }
            mark(3);
            cg_wait();  // every CTA finished reading the buffers written below (round R - 1)
            mark(4);
            if (rot) {
                double bf[KF][NB8];
#pragma unroll
                for (int kf = 0; kf < KF; ++kf)
#pragma unroll
                    for (int ct = 0; ct < NB8; ++ct) bf[kf][ct] = Jb[(4 * kf + lc) * JP + ct * 8 + lr];
                for (int sl0 = 2 * warp; sl0 < Mp / 8; sl0 += 16) {  // Mp / 8 is a multiple of 4
                    double af[2][KF];
#pragma unroll
                    for (int u = 0; u < 2; ++u)
#pragma unroll
                        for (int kf = 0; kf < KF; ++kf) af[u][kf] = Ws[(4 * kf + lc) * P + (sl0 + u) * 8 + lr];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
#pragma unroll
                        for (int ct = 0; ct < NB8; ++ct) {
                            double o0 = 0.0, o1 = 0.0;
#pragma unroll
                            for (int kf = 0; kf < KF; ++kf) jac_dmma(o0, o1, af[u][kf], bf[kf][ct]);
                            // o0 = out[lr][2lc], o1 = out[lr][2lc + 1]: trade with
                            // lane ^ 4 so each lane holds two rows of one column
                            const bool ev = (lr & 1) == 0;
                            const double y = __shfl_xor_sync(0xffffffffu, ev ? o1 : o0, 4);
                            const int cc = 2 * lc + (ev ? 0 : 1), row = (sl0 + u) * 8 + (lr & ~1);
                            cg_st_async(dst[ct] + unsigned((cc * P + row) * 8), ev ? o0 : y, ev ? y : o1, dbar[ct]);
                        }
                    }
                }
            } else {
                for (int e = 2 * t; e < C2 * Mp; e += 2 * blockDim.x) {
                    const int c = e / Mp, i = e % Mp, h = c / BW, cc = c % BW;
                    cg_st_async(dst[h] + unsigned((cc * P + i) * 8), Ws[size_t(c) * P + i], Ws[size_t(c) * P + i + 1],
                                dbar[h]);
                }
            }
            if (rot && t == 0)
                asm volatile("st.shared::cluster.u32 [%0], %1;\n" ::"r"(cg_map(&sflag[sweep & 1], 0)), "r"(1u)
                             : "memory");
            if (r == 0 && g == 0 && t == 0) sflag[(sweep + 1) & 1] = 0u;  // read by all at the end of sweep - 1
            __syncthreads();
            mark(5);
            if (r == nb - 1)
                cg_arrive_release();  // the sweep's flag stores, for the read below
            else
                cg_arrive_relaxed();
            mark(6);
        }
        cg_wait();
        if (t == 0) {
            unsigned v;
            asm volatile("ld.shared::cluster.u32 %0, [%1];\n" : "=r"(v) : "r"(cg_map(&sflag[sweep & 1], 0)) : "memory");
            s_stop = v == 0u;
        }
        cg_arrive_relaxed();
        __syncthreads();
        ++sweep;
        if (s_stop || n < 2) break;
    }
    cg_wait();
    // the resident pair (round 0's) back to W once its last columns arrived
    if (t == 0 && R > 0) jb_mbar_wait(&inbar[R & 1], unsigned((R - 1) >> 1) & 1u);
    __syncthreads();
    {
        int bI, bJ;
        pair_of(g, 0, bI, bJ);
        const double* Ws = Wb0 + size_t(R & 1) * C2 * P;
        for (int e = t; e < C2 * m; e += blockDim.x) {
            const int c = e / m, i = e % m;
            const int gc = c < BW ? bI * BW + c : bJ * BW + (c - BW);
            if (gc < n) a.W[i + int64_t(gc) * a.ldw] = Ws[size_t(c) * P + i];
        }
    }
    for (int e = t; e < kCgVRows * n; e += blockDim.x) {
        const int c = e / kCgVRows, i = e % kCgVRows;
        if (vr0 + i < n) a.V[(vr0 + i) + int64_t(c) * a.ldv] = Vs[c * kCgVP + i];
    }
    if (g == 0 && t == 0) {
        a.flags[4] = sweep;
        if (econv) a.flags[3] = RLRA_ECONV;
    }
    if (clk)
        for (int i = 0; i < 7; ++i) a.phase_clk[i] = ph[i];
}

__device__ __forceinline__ void sg_cp16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(jb_smem(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void sg_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void sg_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ----------------------- streaming Gram block Jacobi, 48-column pairs -------
// For l x l inputs too tall for shared memory (the C2 R-hat, 6100 x 6100):
// blocks of 24 columns so the nb/2 = 128 pair CTAs cover most SMs (blocks of
// 32 leave 52 idle), the cross/intra cyclic schedule of bgram_jacobi_kernel
// (every column pair once per sweep), point-to-point block versions instead
// of a grid barrier per round.  W and V are the engine's own padded copies
// (small_svd_tall): leading dimensions a multiple of kSCR rows, columns
// padded to nb * kSGB, padding zero, so every chunk of a pair is 48 full
// columns of kSCR doubles.  Per visit the chunks (64 rows x 48 columns) stream
// through a kSNST-stage shared-memory ring filled by cp.async (16 bytes per
// thread request, 6 per thread per chunk: 1-D bulk copies of 512 B measured
// 1.65x slower), kSNST - 1 chunks in flight while the 8 warps work on one; the
// sequence is: the Gram's chunks of W_p, then (speculatively, issued while
// the Gram's tail and the rotation steps run) W_p's chunks again for W_p J,
// then V_p's for V_p J (drained unused when nothing rotated).
//   1. G = W_p^T W_p: each warp a k-slice of every chunk for all 21 upper 8x8
//      tiles (registers), the 8 partial Grams summed in a fixed order;
//   2. the visit's steps on G: the 24 pair rotations (reference formula and
//      skip rule, branch-free fast form) then every thread updates its 2x2
//      pair blocks of G (double-buffered) and J — two barriers per step;
//   3. W_p J and V_p J on DMMA (16 x 24 warp tiles), written straight out.
// A visit whose blocks are unchanged since the pair's last rotation-free
// visit is skipped exactly (same Gram bits, again no rotation).
constexpr int kSGB = 24, kSC2 = 48, kSNB8 = 6, kSNT = 21, kSCR = 64, kSNST = 4;
constexpr int kSCP = kSCR + 4;   // chunk pitch (== 4 mod 16), 16-byte aligned rows
constexpr int kSGP = kSC2 + 1;   // G / J pitch
constexpr int kSJP = kSC2 + 4;   // J pitch for B fragments (== 4 mod 16)
constexpr int kSPT = 7;          // tiles per partial-Gram reduction round (3 rounds of 7)
constexpr int kSXG = kSC2 * (kSC2 + 1) / 2;  // packed upper triangle of a 48 x 48 partial Gram
// packed row-major upper triangle: row i starts at sx_off(i) = i*48 - i(i-1)/2
__device__ __forceinline__ int sx_off(int i) { return i * kSC2 - (i * (i - 1)) / 2; }

constexpr size_t kSGramSmem = sizeof(double) * (size_t(kSNST) * kSC2 * kSCP + size_t(8) * kSPT * 64 +
                                                3 * kSC2 * kSGP + kSC2 * kSJP + 2 * kSGB);

__global__ void __launch_bounds__(256, 1) sgram_jacobi_kernel(GramJacArgs a) {
    extern __shared__ __align__(16) double ssm[];
    double* Ring = ssm;                        // kSNST stages: 48 columns x kSCR rows, pitch kSCP
    double* Pb = Ring + kSNST * kSC2 * kSCP;   // 8 warps x kSPT tiles x 64 partial Grams
    double* G0 = Pb + 8 * kSPT * 64;           // two 48 x 49 buffers
    double* J = G0 + 2 * kSC2 * kSGP;          // 48 x 49
    double* Jb = J + kSC2 * kSGP;              // 48 x 52
    double* rc = Jb + kSC2 * kSJP;             // per pair: c, s
    double* rs = rc + kSGB;
    __shared__ int rpq[kSGB];
    __shared__ int s_skip;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31, lr = lane >> 2, lc = lane & 3;
    const int m = a.m, n = a.n, nb = a.nb, np = nb / 2;
    const int ncw = int(a.ldw / kSCR), ncv = int(a.ldv / kSCR);  // chunks of W / V columns
    const int H = a.halves ? 2 : 1;  // tasks per visit (row halves)
    auto prog = [&](unsigned code, unsigned task, unsigned R) {  // RLRA_SGRAM_DEBUG progress record
        if (a.dbg && threadIdx.x == 0) {
            a.dbg[16 + 4 * blockIdx.x] = code;
            a.dbg[17 + 4 * blockIdx.x] = task;
            a.dbg[18 + 4 * blockIdx.x] = R;
        }
    };
    volatile int* flags = a.flags;
    __shared__ int s_task;
    // ring counters (identical in every thread): qn chunks issued (one
    // cp.async group each), qu consumed; chunk q uses stage q % kSNST
    unsigned qn = 0, qu = 0;
    int sweep = 0;
    for (;;) {
        if (sweep >= kOneSidedSweepCap) {
            if (blockIdx.x == 0 && t == 0) flags[3] = RLRA_ECONV;
            break;
        }
        if (blockIdx.x == 0 && t == 0) flags[(sweep + 1) % 3] = 0;
        // dynamic schedule: CTAs take the sweep's (round, pair) visits in
        // order from a counter, so a CTA whose visit was cheap (nothing
        // rotated, or skipped) runs ahead into the next round's ready pairs
        // instead of idling until its fixed pair slot's inputs arrive.  Every
        // visit with a smaller index is held by a running CTA, so the version
        // waits below always resolve.
        for (;;) {
            {
                if (t == 0) s_task = int(atomicAdd(a.tasks + sweep, 1u));
                __syncthreads();
                // (every path passes the s_skip barrier below before thread 0
                // can write s_task again, so no second barrier is needed here)
                const int task = s_task;
                prog(1, task, 0);
                if (task >= nb * np * H) break;
                const int hh = task % H;  // the row half this task covers (halves mode)
                const int r = (task / H) / np, g = (task / H) % np;
                // halves: chunks [cbeg, cbeg + nch) of the W rows; the two tasks
                // of a visit are adjacent in the order, so a half waiting on its
                // partner's partial Gram always has the partner held or next
                const int nch2 = (ncw + 1) / 2;
                const int cbeg = H == 2 ? hh * nch2 : 0;
                const int nch = H == 2 ? min(ncw, cbeg + nch2) - cbeg : ncw;
                unsigned* verv = a.ver + hh * nb;  // this half's block versions
                const unsigned R = unsigned(sweep) * unsigned(nb) + unsigned(r);  // the visit's global round
                const bool intra = r == nb - 1;
                int bI = 2 * g, bJ = 2 * g + 1;
                if (!intra) {
                    const int b1 = rr_col(g, r, nb), b2 = rr_col(nb - 1 - g, r, nb);
                    bI = min(b1, b2);
                    bJ = max(b1, b2);
                }
                auto gcol = [&](int c) { return c < kSGB ? bI * kSGB + c : bJ * kSGB + (c - kSGB); };
                const int pid = intra ? nb * nb + g : bI * nb + bJ;
                const int xslot = int(R & 1u) * np + g;  // partial-Gram slot (two generations)
                if (t == 0) {
                    sg_wait_dbg(verv + bI, R, a.dbg, 1, R, hh);
                    sg_wait_dbg(verv + bJ, R, a.dbg, 2, R, hh);
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire the previous writers' stores
                    // (halves: both tasks decide alike — clean and mod only change
                    // after both halves' partial Grams were exchanged)
                    const unsigned c = __ldcg(a.clean + pid);
                    s_skip = c != 0u && c >= __ldcg(a.mod + bI) && c >= __ldcg(a.mod + bJ);
                    if (hh == 0) {
                        atomicAdd(a.counters + 0, 1ull);
                        if (s_skip) atomicAdd(a.counters + 1, 1ull);
                    }
                }
                prog(2, 0, R);
                __syncthreads();
                if (s_skip) {
                    if (t == 0) {
                        if (H == 2) {
                            // the slot's next user may write — but only once this
                            // half's previous use of the slot (round R - 2) was read:
                            // a skipped visit must not overtake it (acks stay monotone)
                            if (R >= 2u) sg_wait_dbg(a.xack + 2 * xslot + hh, R - 1, a.dbg, 5, R, hh);
                            jb_publish(a.xack + 2 * xslot + hh, R + 1);
                        }
                        // nothing written: the fence after the version waits orders
                        // the predecessors' W writes before these stores
                        jb_store_relaxed(verv + bI, R + 1);
                        jb_store_relaxed(verv + bJ, R + 1);
                    }
                    continue;
                }
                // the visit's chunk sequence: [0, ncw) Gram of W, [ncw, 2 ncw)
                // W for the apply, [2 ncw, 2 ncw + ncv) V for the apply (issued
                // only once the pair's V blocks are current, see step 3)
                int kend = 2 * nch;
                int kin = 0;  // next sequence position to issue
                auto issue = [&]() {  // sequence position kin into stage qn % kSNST (all threads)
                    const int k = kin;
                    const bool isv = k >= 2 * nch;
                    const double* X = isv ? a.V : a.W;
                    const int64_t ld = isv ? a.ldv : a.ldw;
                    const int row0 = (isv ? k - 2 * nch : cbeg + (k < nch ? k : k - nch)) * kSCR;
                    double* dst = Ring + (qn % kSNST) * (kSC2 * kSCP);
#pragma unroll
                    for (int it = 0; it < kSC2 * kSCR / 2 / 256; ++it) {  // 16-byte pieces: 32 per column
                        const int e = t + 256 * it, c = e >> 5, r2 = (e & 31) * 2;
                        sg_cp16(dst + c * kSCP + r2, X + row0 + r2 + int64_t(gcol(c)) * ld);
                    }
                };
                for (; qn - qu < unsigned(kSNST - 1) && kin < kend; ++qn, ++kin) {
                    issue();
                    sg_commit();
                }
                // consume the next chunk: wait for its group (kSNST - 2 younger
                // groups may stay in flight), run body on its stage, then refill
                // the ring (the stage of chunk qn - kSNST = qu - 1, released by the
                // barrier) kSNST - 1 chunks ahead; an empty group keeps the
                // group count aligned at the sequence's end
                // (the barrier after the wait also retires every thread's reads of
                // chunk q - 1's stage, the one refilled below)
                auto consume = [&](auto&& body) {
                    const unsigned q = qu++;
                    if (qn - qu >= unsigned(kSNST - 2)) sg_wait<kSNST - 2>(); else sg_wait<0>();
                    __syncthreads();
                    body(Ring + (q % kSNST) * (kSC2 * kSCP));
                    if (kin < kend) {
                        issue();
                        ++qn;
                        ++kin;
                    }
                    sg_commit();
                };
                // ---- 1. Gram -------------------------------------------------
                {
                    double acc[kSNT][2];
#pragma unroll
                    for (int u = 0; u < kSNT; ++u) acc[u][0] = acc[u][1] = 0.0;
                    for (int ch = 0; ch < nch; ++ch) {
                        consume([&](const double* Cb) {
#pragma unroll
                            for (int h = 0; h < kSCR / 32; ++h) {
                                const int kk = (warp + 8 * h) * 4;
                                double f[kSNB8];
#pragma unroll
                                for (int bb = 0; bb < kSNB8; ++bb) f[bb] = Cb[(bb * 8 + lr) * kSCP + kk + lc];
                                int u = 0;
#pragma unroll
                                for (int bi = 0; bi < kSNB8; ++bi)
#pragma unroll
                                    for (int bj = bi; bj < kSNB8; ++bj, ++u)
                                        jac_dmma(acc[u][0], acc[u][1], f[bi], f[bj]);
                            }
                        });
                    }
                    // the 8 warps' partials summed in a fixed order, kSPT tiles a round
#pragma unroll
                    for (int u0 = 0; u0 < kSNT; u0 += kSPT) {
#pragma unroll
                        for (int u = u0; u < u0 + kSPT; ++u) {
                            Pb[(warp * kSPT + (u - u0)) * 64 + lr * 8 + 2 * lc] = acc[u][0];
                            Pb[(warp * kSPT + (u - u0)) * 64 + lr * 8 + 2 * lc + 1] = acc[u][1];
                        }
                        __syncthreads();
                        for (int e = t; e < kSPT * 64; e += 256) {
                            const int u = u0 + (e >> 6), w = e & 63;
                            int bi = 0, rem = u;
                            while (rem >= kSNB8 - bi) rem -= kSNB8 - bi++;
                            const int bj = bi + rem;
                            double sum = 0.0;
#pragma unroll
                            for (int ww = 0; ww < 8; ++ww) sum += Pb[(ww * kSPT + (u - u0)) * 64 + w];
                            const int row = bi * 8 + (w >> 3), col = bj * 8 + (w & 7);
                            G0[row * kSGP + col] = sum;
                            G0[col * kSGP + row] = sum;
                        }
                        __syncthreads();
                    }
                    if (H == 2) {
                        // exchange the halves' partial Grams (upper triangle,
                        // row-major packed): wait until the slot's previous user
                        // (round R - 2) read our last partial, write ours, then
                        // read the partner's; G = P + P' is the same sum in both
                        // halves (IEEE addition commutes), so both run the same steps
                        double* mine = a.xg + (size_t(xslot) * 2 + hh) * kSXG;
                        const double* theirs = a.xg + (size_t(xslot) * 2 + (1 - hh)) * kSXG;
                        prog(3, 0, R);
                        if (t == 0 && R >= 2u) {
                            sg_wait_dbg(a.xack + 2 * xslot + (1 - hh), R - 1, a.dbg, 3, R, hh);
                            asm volatile("fence.acq_rel.gpu;" ::: "memory");
                        }
                        __syncthreads();
                        for (int e = t; e < kSC2 * kSC2; e += 256) {
                            const int i = e / kSC2, j = e % kSC2;
                            if (j >= i) __stcg(mine + sx_off(i) + (j - i), G0[i * kSGP + j]);
                        }
                        __syncthreads();
                        prog(4, 0, R);
                        if (t == 0) {
                            __threadfence();
                            jb_publish(a.xstamp + 2 * xslot + hh, R + 1);
                            sg_wait_dbg(a.xstamp + 2 * xslot + (1 - hh), R + 1, a.dbg, 4, R, hh);
                            asm volatile("fence.acq_rel.gpu;" ::: "memory");
                        }
                        __syncthreads();
                        for (int e = t; e < kSC2 * kSC2; e += 256) {
                            const int i = e / kSC2, j = e % kSC2;
                            if (j < i) continue;
                            const double v = G0[i * kSGP + j] + __ldcg(theirs + sx_off(i) + (j - i));
                            G0[i * kSGP + j] = v;
                            G0[j * kSGP + i] = v;
                        }
                        __syncthreads();
                        if (t == 0) {
                            __threadfence();
                            jb_publish(a.xack + 2 * xslot + hh, R + 1);
                        }
                    }
                }
                for (int e = t; e < kSC2 * kSC2; e += 256) J[(e / kSC2) * kSGP + e % kSC2] = (e / kSC2 == e % kSC2) ? 1.0 : 0.0;
                __syncthreads();
                // ---- 2. the visit's steps ------------------------------------
                int rot = 0;
                const int nsteps = intra ? kSGB - 1 : kSGB;
                for (int st = 0; st < nsteps; ++st) {
                    const double* Gc = G0 + (st & 1) * kSC2 * kSGP;
                    double* Gn = G0 + ((st & 1) ^ 1) * kSC2 * kSGP;
                    int act = 0;
                    if (t < kSGB) {
                        const int pq = bgram_pair<kSGB>(intra, t, st);
                        const int p = pq & 255, q = pq >> 8;
                        const double pp = Gc[p * kSGP + p], qq = Gc[q * kSGP + q], pqv = Gc[p * kSGP + q];
                        double c, sn;
                        if (!jac_rotation_fast(pp, qq, pqv, c, sn, act)) act = jac_rotation_ref(pp, qq, pqv, c, sn);
                        rc[t] = c;
                        rs[t] = sn;
                        rpq[t] = pq | (act << 16);
                    }
                    rot |= __syncthreads_or(act);
                    for (int b = t; b < kSGB * kSGB; b += 256) {
                        const int k = b / kSGB, l = b % kSGB;
                        const int pqk = rpq[k], pql = rpq[l];
                        const int pk = pqk & 255, qk = (pqk >> 8) & 255, pl = pql & 255, ql = (pql >> 8) & 255;
                        const bool ak = (pqk >> 16) != 0, al = (pql >> 16) != 0;
                        const double ck = rc[k], sk = rs[k], cl = rc[l], sl = rs[l];
                        const double j0 = J[pk * kSGP + pl], j1 = J[pk * kSGP + ql];
                        const double j2 = J[qk * kSGP + pl], j3 = J[qk * kSGP + ql];
                        double b00 = Gc[pk * kSGP + pl], b01 = Gc[pk * kSGP + ql];
                        double b10 = Gc[qk * kSGP + pl], b11 = Gc[qk * kSGP + ql];
                        if (al) {
                            J[pk * kSGP + pl] = cl * j0 - sl * j1;
                            J[pk * kSGP + ql] = sl * j0 + cl * j1;
                            J[qk * kSGP + pl] = cl * j2 - sl * j3;
                            J[qk * kSGP + ql] = sl * j2 + cl * j3;
                        }
                        {  // branch-free (selects keep the values of a skipped rotation)
                            const double x0 = cl * b00 - sl * b01, x1 = sl * b00 + cl * b01;
                            const double x2 = cl * b10 - sl * b11, x3 = sl * b10 + cl * b11;
                            b00 = al ? x0 : b00, b01 = al ? x1 : b01, b10 = al ? x2 : b10, b11 = al ? x3 : b11;
                            const double y0 = ck * b00 - sk * b10, y2 = sk * b00 + ck * b10;
                            const double y1 = ck * b01 - sk * b11, y3 = sk * b01 + ck * b11;
                            b00 = ak ? y0 : b00, b01 = ak ? y1 : b01, b10 = ak ? y2 : b10, b11 = ak ? y3 : b11;
                        }
                        if (k <= l) {
                            Gn[pk * kSGP + pl] = b00;
                            Gn[pk * kSGP + ql] = b01;
                            Gn[qk * kSGP + pl] = b10;
                            Gn[qk * kSGP + ql] = b11;
                            Gn[pl * kSGP + pk] = b00;
                            Gn[ql * kSGP + pk] = b01;
                            Gn[pl * kSGP + qk] = b10;
                            Gn[ql * kSGP + qk] = b11;
                        }
                    }
                    __syncthreads();
                }
                prog(6, rot, R);
                if (rot) {
                    if (t == 0) flags[sweep % 3] = 1;
                    for (int e = t; e < kSC2 * kSC2; e += 256) Jb[(e / kSC2) * kSJP + e % kSC2] = J[(e / kSC2) * kSGP + e % kSC2];
                    __syncthreads();
                    // ---- 3. W_p J, V_p J: warp (wr, wc) owns rows wr*16..+16, cols wc*24..+24 of a chunk
                    const int wr = warp & 3, wc = warp >> 2;
                    int ocol[3][2];
#pragma unroll
                    for (int ct = 0; ct < 3; ++ct)
#pragma unroll
                        for (int h = 0; h < 2; ++h) ocol[ct][h] = gcol(wc * 24 + ct * 8 + 2 * lc + h);
                    double bf[kSC2 / 4][3];
#pragma unroll
                    for (int kf = 0; kf < kSC2 / 4; ++kf)
#pragma unroll
                        for (int ct = 0; ct < 3; ++ct) bf[kf][ct] = Jb[(4 * kf + lc) * kSJP + wc * 24 + ct * 8 + lr];
                    __shared__ unsigned s_tick[2];
                    for (int mat = 0; mat < 2; ++mat) {
                        double* X = mat == 0 ? a.W : a.V;
                        const int64_t ld = mat == 0 ? a.ldw : a.ldv;
                        const int rows = mat == 0 ? m : n;
                        const int nchm = mat == 0 ? nch : ncv;
                        if (mat == 1) {
                            // W_p J is out: publish W now, so the blocks' next
                            // owners start their Grams while this CTA does V_p J.
                            // V keeps its own order: this pair's V update is the
                            // s_tick-th of each block; wait for the earlier ones
                            __syncthreads();
                            if (t == 0) {
                                s_tick[0] = __ldcg(a.vtick + bI);
                                s_tick[1] = __ldcg(a.vtick + bJ);
                                if (!a.skip_v) {
                                    __stcg(a.vtick + bI, s_tick[0] + 1u);
                                    __stcg(a.vtick + bJ, s_tick[1] + 1u);
                                }
                                __stcg(a.mod + bI, R + 1u);
                                __stcg(a.mod + bJ, R + 1u);
                                if (hh == 0) {
                                    atomicAdd(a.counters + 2, 1ull);
                                    if (a.phase_clk) atomicAdd(reinterpret_cast<unsigned long long*>(a.phase_clk) + 2 * sweep + 1, 1ull);
                                }
                                __threadfence();
                                jb_store_relaxed(verv + bI, R + 1);
                                jb_store_relaxed(verv + bJ, R + 1);
                                if (!a.skip_v) {
                                    jb_wait_at_least(a.vdone + bI, s_tick[0]);
                                    jb_wait_at_least(a.vdone + bJ, s_tick[1]);
                                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                                }
                            }
                            __syncthreads();
                            if (a.skip_v) break;  // W only: the ring is empty (every W chunk consumed)
                            kend = 2 * nch + ncv;
                            for (; qn - qu < unsigned(kSNST - 1) && kin < kend; ++qn, ++kin) {
                                issue();
                                sg_commit();
                            }
                        }
                        for (int ch = 0; ch < nchm; ++ch) {
                            const int k0 = ((mat == 0 ? cbeg : 0) + ch) * kSCR;
                            consume([&](const double* Cb) {
                                double o[2][3][2];
#pragma unroll
                                for (int f = 0; f < 2; ++f)
#pragma unroll
                                    for (int ct = 0; ct < 3; ++ct) o[f][ct][0] = o[f][ct][1] = 0.0;
#pragma unroll
                                for (int kf = 0; kf < kSC2 / 4; ++kf) {
                                    double af[2];
#pragma unroll
                                    for (int f = 0; f < 2; ++f) af[f] = Cb[(4 * kf + lc) * kSCP + wr * 16 + f * 8 + lr];
#pragma unroll
                                    for (int f = 0; f < 2; ++f)
#pragma unroll
                                        for (int ct = 0; ct < 3; ++ct)
                                            jac_dmma(o[f][ct][0], o[f][ct][1], af[f], bf[kf][ct]);
                                }
#pragma unroll
                                for (int f = 0; f < 2; ++f) {
                                    const int row = k0 + wr * 16 + f * 8 + lr;
                                    if (row >= rows) continue;
#pragma unroll
                                    for (int ct = 0; ct < 3; ++ct)
#pragma unroll
                                        for (int h = 0; h < 2; ++h)
                                            if (ocol[ct][h] < n) X[row + int64_t(ocol[ct][h]) * ld] = o[f][ct][h];
                                }
                            });
                        }
                    }
                    __syncthreads();
                    if (t == 0 && !a.skip_v) {
                        __threadfence();
                        jb_publish(a.vdone + bI, s_tick[0] + 1u);
                        jb_publish(a.vdone + bJ, s_tick[1] + 1u);
                    }
                } else {
                    // nothing rotated: drain the speculatively issued apply chunks
                    // (the rest of the sequence is never issued)
                    sg_wait<0>();
                    qu = qn;
                }
                __syncthreads();
                if (t == 0 && !rot) {  // (a rotating visit published W before its V update)
                    __stcg(a.clean + pid, R + 1u);
                    __threadfence();
                    jb_store_relaxed(verv + bI, R + 1);
                    jb_store_relaxed(verv + bJ, R + 1);
                }
            }
        }
        prog(8, sweep, 0);
        grid_sync(a.bar);
        prog(9, sweep, 0);
        if (a.phase_clk && blockIdx.x == 0 && t == 0) {  // RLRA_JACOBI_PHASES: sweep end times
            unsigned long long tn;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
            a.phase_clk[2 * sweep] = (long long)tn;
        }
        const int rotated = flags[sweep % 3];
        ++sweep;
        if (!rotated || n < 2) break;
    }
    if (blockIdx.x == 0 && t == 0) flags[4] = sweep;
}

int coop_grid(Context& ctx, const void* kern, int want_blocks) {
    int per_sm = 0;
    RLRA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kJacThreads, 0));
    const int cap = std::max(1, per_sm) * ctx.num_sms;
    return std::max(1, std::min(want_blocks, cap));
}

// ---------------------------------------------------- two-sided Jacobi ---
struct TwoSidedArgs {
    unsigned* bar;  // grid_sync state (Context::gbar)
    double* M;
    int64_t ldm;
    int n;
    double* U;
    int64_t ldu;
    double* cs;      // per-pair (c, s, active) triples: 3 * n2/2
    double* part;    // per-block partials for the off-diagonal norm
    double tnorm;
    int* status;
};

__global__ void __launch_bounds__(kJacThreads) twosided_jacobi_kernel(TwoSidedArgs a) {
    __shared__ double sh[32];
    const int n = a.n, n2 = n + (n & 1);
    const int gt = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    int sweep = 0;
    const double thr = 1e-14 * fmax(a.tnorm, 1e-300);  // reference jacobi.hpp:99
    for (;;) {
        if (n <= 1) break;
        // off-diagonal norm sqrt(sum_{i<j} 2 M_ij^2), fixed order
        double v = 0.0;
        for (int64_t e = gt; e < int64_t(n) * n; e += nt) {
            const int i = int(e % n), j = int(e / n);
            if (i < j) {
                const double x = a.M[i + int64_t(j) * a.ldm];
                v += 2.0 * x * x;
            }
        }
        v = block_sum_fixed(v, sh);
        if (threadIdx.x == 0) a.part[blockIdx.x] = v;
        grid_sync(a.bar);
        double off = 0.0;
        for (int b = 0; b < int(gridDim.x); ++b) off += a.part[b];
        off = sqrt(off);
        grid_sync(a.bar);
        if (!(off > thr)) break;
        if (sweep++ >= kTwoSidedSweepCap) {
            if (gt == 0) *a.status = RLRA_ECONV;
            break;
        }
        for (int r = 0; r < n2 - 1; ++r) {
            // angles for every disjoint pair of this round from the current M
            for (int pi = gt; pi < n2 / 2; pi += nt) {
                const int ca = rr_col(pi, r, n2), cb = rr_col(n2 - 1 - pi, r, n2);
                const int p = min(ca, cb), q = max(ca, cb);
                double c = 1.0, s = 0.0, act = 0.0;
                if (q < n) {
                    const double apq = a.M[p + int64_t(q) * a.ldm];
                    if (fabs(apq) > 1e-300) {
                        const double theta =
                            (a.M[q + int64_t(q) * a.ldm] - a.M[p + int64_t(p) * a.ldm]) / (2.0 * apq);
                        const double t = (theta >= 0.0 ? 1.0 : -1.0) /
                                         (fabs(theta) + sqrt(1.0 + theta * theta));
                        c = 1.0 / sqrt(1.0 + t * t);
                        s = t * c;
                        act = 1.0;
                    }
                }
                a.cs[3 * pi] = c;
                a.cs[3 * pi + 1] = s;
                a.cs[3 * pi + 2] = act;
            }
            grid_sync(a.bar);
            // columns of M and U
            for (int64_t e = gt; e < int64_t(n2 / 2) * n; e += nt) {
                const int pi = int(e / n), i = int(e % n);
                if (a.cs[3 * pi + 2] == 0.0) continue;
                const int ca = rr_col(pi, r, n2), cb = rr_col(n2 - 1 - pi, r, n2);
                const int p = min(ca, cb), q = max(ca, cb);
                const double c = a.cs[3 * pi], s = a.cs[3 * pi + 1];
                double* mp = a.M + int64_t(p) * a.ldm;
                double* mq = a.M + int64_t(q) * a.ldm;
                const double xp = mp[i], xq = mq[i];
                mp[i] = c * xp - s * xq;
                mq[i] = s * xp + c * xq;
                double* up = a.U + int64_t(p) * a.ldu;
                double* uq = a.U + int64_t(q) * a.ldu;
                const double yp = up[i], yq = uq[i];
                up[i] = c * yp - s * yq;
                uq[i] = s * yp + c * yq;
            }
            grid_sync(a.bar);
            // rows of M
            for (int64_t e = gt; e < int64_t(n2 / 2) * n; e += nt) {
                const int pi = int(e / n), i = int(e % n);
                if (a.cs[3 * pi + 2] == 0.0) continue;
                const int ca = rr_col(pi, r, n2), cb = rr_col(n2 - 1 - pi, r, n2);
                const int p = min(ca, cb), q = max(ca, cb);
                const double c = a.cs[3 * pi], s = a.cs[3 * pi + 1];
                const double xp = a.M[p + int64_t(i) * a.ldm], xq = a.M[q + int64_t(i) * a.ldm];
                a.M[p + int64_t(i) * a.ldm] = c * xp - s * xq;
                a.M[q + int64_t(i) * a.ldm] = s * xp + c * xq;
            }
            grid_sync(a.bar);
        }
    }
}

__global__ void diag_of_kernel(const double* M, int64_t ldm, int n, double* d) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        d[i] = M[i + int64_t(i) * ldm];
}

__global__ void eig_scatter_kernel(const double* d, const int* rank, const double* U, int64_t ldu,
                                   int n, double* values, double* vec, int64_t ldv) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(n) * n;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int j = int(e / n), i = int(e % n);
        const int r = rank[j];
        vec[i + int64_t(r) * ldv] = U[i + int64_t(j) * ldu];
        if (i == 0) values[r] = d[j];
    }
}

__global__ void asym_kernel(const double* T, int64_t ldt, int n, double* part) {
    __shared__ double sh[32];
    double v = 0.0;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(n) * n;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e % n), j = int(e / n);
        if (i < j) v = fmax(v, fabs(T[i + int64_t(j) * ldt] - T[j + int64_t(i) * ldt]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t = fmax(t, sh[w]);
        part[blockIdx.x] = t;
    }
}

}  // namespace

// cluster launch of cgram_jacobi_kernel<8>: np = nb / 2 CTAs, one cluster
cudaLaunchConfig_t cgram_config(Context& ctx, int np, size_t smem, cudaLaunchAttribute* attr) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(np));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx.stream;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(np);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cfg;
}

void cgram_attrs(size_t smem) {
    static size_t set = 0;
    if (set < smem) {
        RLRA_CUDA(cudaFuncSetAttribute(cgram_jacobi_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        RLRA_CUDA(cudaFuncSetAttribute(cgram_jacobi_kernel<8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        set = smem;
    }
}

// can one cluster of np CTAs with this shared memory be resident?
bool cgram_fits(Context& ctx, int np, size_t smem) {
    static const bool off = std::getenv("RLRA_CGRAM_OFF") != nullptr;
    if (off || np < 2 || np > 16) return false;
    cgram_attrs(smem);
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = cgram_config(ctx, np, smem, attr);
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, (void*)cgram_jacobi_kernel<8>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return nclusters >= 1;
}

// false when the cluster cannot be placed at launch time (e.g. another
// context holds the SMs of every GPC): the caller takes the L2 variant
bool launch_cgram(Context& ctx, const CGramArgs& c, size_t smem) {
    cgram_attrs(smem);
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = cgram_config(ctx, c.nb / 2, smem, attr);
    if (cudaLaunchKernelEx(&cfg, cgram_jacobi_kernel<8>, c) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return true;
}

// E = V^T V - I over the upper triangle (E from an upper-tiles-only Gram):
// the diagonal shifted in place, per-CTA max |E_ij| (NaN counts as infinite)
__global__ void orth_defect_kernel(double* E, int64_t lde, int n, double* part) {
    __shared__ double red[256];
    double mx = 0.0;
    for (int j = blockIdx.x; j < n; j += gridDim.x)
        for (int i = threadIdx.x; i <= j; i += blockDim.x) {
            double e = E[i + int64_t(j) * lde];
            if (i == j) {
                e -= 1.0;
                E[i + int64_t(j) * lde] = e;
            }
            const double a = fabs(e);
            mx = (a == a) ? fmax(mx, a) : INFINITY;
        }
    red[threadIdx.x] = mx;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// V from the rotated W of an upper-triangular square R: the one-sided
// rotations keep W = R V, so V = R^{-1} W (blocked back substitution on
// DMMA).  This is accurate when R's column-scaled condition is modest (the
// QR-preconditioned Jacobi SVD of Drmac-Veselic; R-hat of a QB or rsvd is
// graded by construction), so it is verified, not assumed: accepted when
// max|V^T V - I| <= kVsolveTol; a defect above kVsolveExact (the level the
// accumulated rotations reach at l ~ 10^4: 1.6e-13 at C2) gets one
// Newton-Schulz step V <- V - V E / 2, taking it to O(E^2) + rounding.  Returns false
// (V garbage) when rejected; the caller re-runs the sweeps accumulating V.
constexpr double kVsolveTol = 1e-11, kVsolveExact = 1e-12;
bool vsolve_from_r(Context& ctx, const DMat& Rm, const DMat& W, const DMat& V, double* defect) {
    const int n = int(Rm.rows);
    ProfScope prof(ctx, "svd_vsolve", n, n, 0, 0.0);
    copy_mat(ctx, W, V);
    upper_tri_solve_inplace(ctx, Rm, V, true);
    DMatBuf E(ctx, n, n);
    GemmOpts sy;
    sy.upper_tiles_only = true;
    gemm(ctx, Op::T, Op::N, 1.0, V, V, 0.0, E, sy);
    const int blocks = std::min(n, ctx.num_sms);
    Buf part(ctx, sizeof(double) * blocks);
    orth_defect_kernel<<<blocks, 256, 0, ctx.stream>>>(E.m.p, E.m.ld, n, part.d());
    RLRA_LAUNCH_CHECK();
    ++ctx.launches;
    std::vector<double> h(blocks);
    RLRA_CUDA(cudaMemcpyAsync(h.data(), part.p, sizeof(double) * blocks, cudaMemcpyDeviceToHost, ctx.stream));
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    double mx = 0.0;
    for (double v : h) mx = (v == v) ? std::max(mx, v) : INFINITY;
    *defect = mx;
    // RLRA_SVD_VSOLVE_TOL overrides the acceptance bound (a negative value
    // rejects every solve: the fallback's test hook)
    static const double tol = std::getenv("RLRA_SVD_VSOLVE_TOL") ? std::atof(std::getenv("RLRA_SVD_VSOLVE_TOL"))
                                                                 : kVsolveTol;
    if (!(mx <= tol)) return false;
    static const bool force_ns = std::getenv("RLRA_SVD_VSOLVE_NS") != nullptr;  // test hook
    if (mx <= kVsolveExact && !force_ns) return true;  // already as orthonormal as accumulated rotations
    symmetrize_upper(ctx, E);
    DMatBuf V0(ctx, n, n);
    copy_mat(ctx, V, V0);
    gemm(ctx, Op::N, Op::N, -0.5, V0, E, 1.0, V);
    return true;
}

void small_svd_tall(Context& ctx, const DMat& A, const DMat& U, double* sigma, const DMat& Vout, bool upper_tri) {
    const int m = int(A.rows), n = int(A.cols);
    if (n == 0) return;
    ProfScope prof(ctx, "small_svd", m, n, 0, 0.0);
    // kernel choice: the shared-memory-resident Gram block Jacobi when a
    // block pair fits (l up to ~1400), else the streaming Gram variant;
    // RLRA_SVD_KERNEL=bgram|block|sgram|gram|onesided forces one (A/B timing)
    static const int forced = [] {
        const char* e = std::getenv("RLRA_SVD_KERNEL");
        if (!e) return 0;
        const std::string v(e);
        return v == "bgram" ? 1 : v == "block" ? 2 : v == "sgram" ? 3 : v == "onesided" ? 4 : v == "gram" ? 5
             : v == "cgram" ? 6 : 0;
    }();
    constexpr size_t kSmemCap = 220 * 1024;
    // blocks of 8 columns: twice the CTAs of 16-column blocks, and the
    // per-visit L2 traffic is what bounds a round (l = 510: 12.5 vs 15.0 ms;
    // 4-column blocks: 15.1 ms).  RLRA_BGRAM_BW=16 selects 16.
    static const int bw_env = std::getenv("RLRA_BGRAM_BW") ? std::atoi(std::getenv("RLRA_BGRAM_BW")) : 0;
    int bgw = (n > 16 && bgram_smem<8>(m) <= kSmemCap) ? 8 : 0;
    if (bw_env == 16 && n > 32 && bgram_smem<16>(m) <= kSmemCap) bgw = 16;
    bool use_bgram = (forced == 0 || forced == 1) && bgw > 0;
    // one cluster of pair CTAs when the blocks of 8 fit 16 of them (l <= 256):
    // W stays in shared memory (RLRA_SVD_KERNEL=bgram keeps the L2 variant)
    const int cnb = ceil_div(n, 8) + (ceil_div(n, 8) & 1);
    const bool use_cgram = (forced == 0 || forced == 6) && n > 16 && cnb <= 32 && cgram_smem<8>(m, cnb) <= kSmemCap &&
                           cgram_fits(ctx, cnb / 2, cgram_smem<8>(m, cnb));
    const int snb = ceil_div(n, kSGB) + (ceil_div(n, kSGB) & 1);
    const bool use_sgram = !use_bgram && forced != 2 && forced != 4 && forced != 5 && n > 2 * kSC2 &&
                           snb / 2 <= ctx.num_sms && m >= 2 * kSCR;
    // W's leading dimension even and its pad row zero: bgram stages columns
    // with 16-byte bulk copies; sgram streams whole kSCR-row chunks of
    // snb * kSGB columns, so its W and V are padded to those (zeros)
    const int ldw = use_sgram ? ceil_div(m, kSCR) * kSCR : (m + 1) & ~1;
    const int ldv = use_sgram ? ceil_div(n, kSCR) * kSCR : (n + 1) & ~1;
    const int ncol = use_sgram ? snb * kSGB : n;
    DMatBuf Wb(ctx, ldw, ncol), V(ctx, ldv, ncol);
    RLRA_CUDA(cudaMemsetAsync(Wb.m.p, 0, sizeof(double) * size_t(ldw) * ncol, ctx.stream));
    RLRA_CUDA(cudaMemsetAsync(V.m.p, 0, sizeof(double) * size_t(ldv) * ncol, ctx.stream));
    DMatBuf& W = Wb;
    W.m.rows = m;
    W.m.cols = n;
    V.m.rows = n;
    V.m.cols = n;
    copy_mat(ctx, A, W);
    eye_mat(ctx, V);
    Buf flags(ctx, sizeof(int) * 8), sg(ctx, sizeof(double) * n), rank(ctx, sizeof(int) * n),
        needs(ctx, sizeof(int) * n);
    RLRA_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int) * 8, ctx.stream));
    OneSidedArgs a;
    a.W = W.m.p;
    a.ldw = W.m.ld;
    a.m = m;
    a.n = n;
    a.V = V.m.p;
    a.ldv = V.m.ld;
    a.flags = flags.i();
    if (use_cgram) {
        static const bool want_clk = std::getenv("RLRA_JACOBI_PHASES") != nullptr;
        Buf clkb(ctx, want_clk ? sizeof(long long) * 8 : 8);
        const size_t slots = size_t(2) * cnb * (cnb / 2);
        Buf jlog(ctx, sizeof(double) * slots * 256), rlog(ctx, slots);
        CGramArgs c{W.m.p, W.m.ld, m,     n, cnb, V.m.p, V.m.ld, jlog.d(), static_cast<unsigned char*>(rlog.p), flags.i(),
                    want_clk ? reinterpret_cast<long long*>(clkb.p) : nullptr};
        const bool ok = launch_cgram(ctx, c, cgram_smem<8>(m, cnb));
        if (ok && want_clk) {
            long long h[7];
            RLRA_CUDA(cudaMemcpyAsync(h, clkb.p, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
            RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
            std::fprintf(stderr,
                         "cgram<8> m=%d n=%d clocks: wait_in %lld gram %lld steps %lld jlog %lld cl_wait %lld send %lld "
                         "arrive %lld\n",
                         m, n, h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
        }
        if (ok) goto launched;
    }
    if (use_bgram) {
        GramJacArgs g;
        g.bar = ctx.gbar;
        g.W = W.m.p;
        g.ldw = W.m.ld;
        g.m = m;
        g.n = n;
        g.V = V.m.p;
        g.ldv = V.m.ld;
        g.nb = ceil_div(n, bgw) + (ceil_div(n, bgw) & 1);
        g.flags = flags.i();
        g.inner_cap = 1;
        // V helpers when every pair owner and its helper fit one wave
        static const bool no_help = std::getenv("RLRA_BGRAM_NOHELP") != nullptr;
        g.helpers = (!no_help && g.nb <= ctx.num_sms) ? 1 : 0;
        const size_t nver = size_t(3) * g.nb;
        Buf verb(ctx, sizeof(unsigned) * nver), jb(ctx, g.helpers ? sizeof(double) * g.nb * (2 * bgw) * (2 * bgw) : 8);
        RLRA_CUDA(cudaMemsetAsync(verb.p, 0, sizeof(unsigned) * nver, ctx.stream));
        g.ver = static_cast<unsigned*>(verb.p);
        g.jbuf = jb.d();
        static const bool want_clk = std::getenv("RLRA_JACOBI_PHASES") != nullptr;
        Buf clkb(ctx, want_clk ? sizeof(long long) * 8 : 8);
        g.phase_clk = want_clk ? reinterpret_cast<long long*>(clkb.p) : nullptr;
        void* args[] = {&g};
        const void* kern = bgw == 16 ? (const void*)bgram_jacobi_kernel<16> : (const void*)bgram_jacobi_kernel<8>;
        const size_t smem = bgw == 16 ? bgram_smem<16>(m) : bgram_smem<8>(m);
        RLRA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        const int grid = g.helpers ? g.nb : std::min(g.nb / 2, ctx.num_sms);
        RLRA_CUDA(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(256), args, smem, ctx.stream));
        if (want_clk) {
            long long h[6];
            RLRA_CUDA(cudaMemcpyAsync(h, clkb.p, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
            RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
            std::fprintf(stderr, "bgram<%d> m=%d n=%d clocks: stage %lld gram %lld steps %lld applyW %lld applyV %lld sync %lld\n",
                         bgw, m, n, h[0], h[1], h[2], h[3], h[4], h[5]);
        }
        goto launched;
    }
    {
    constexpr int BW = 8;
    const size_t bj_smem = sizeof(double) * (size_t(2 * BW) * m + 4 * BW * BW);
    const int nblk = ceil_div(n, BW) + (ceil_div(n, BW) & 1);
    int per_sm = 0;
    if (bj_smem <= 200 * 1024 && n > 2 * BW) {
        RLRA_CUDA(cudaFuncSetAttribute(block_jacobi_kernel<BW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(bj_smem)));
        RLRA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, block_jacobi_kernel<BW>, BW * 32,
                                                                bj_smem));
    }
    if (forced != 3 && forced != 4 && forced != 5 && per_sm > 0 && nblk / 2 <= per_sm * ctx.num_sms) {
        BlockJacArgs b;
        b.W = W.m.p;
        b.ldw = W.m.ld;
        b.m = m;
        b.n = n;
        b.V = V.m.p;
        b.ldv = V.m.ld;
        b.nb = nblk;
        b.flags = flags.i();
        b.bar = ctx.gbar;
        void* args[] = {&b};
        RLRA_CUDA(cudaLaunchCooperativeKernel((void*)block_jacobi_kernel<BW>, dim3(nblk / 2), dim3(BW * 32),
                                              args, bj_smem, ctx.stream));
    } else if (use_sgram) {
        // columns too long for shared memory: streaming Gram block Jacobi, 48-column pairs
        static bool attr = false;
        if (!attr) {
            RLRA_CUDA(cudaFuncSetAttribute(sgram_jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(kSGramSmem)));
            attr = true;
        }
        // A = R-hat (upper triangular, square): the sweeps rotate W only and
        // V comes from R^{-1} W afterwards (vsolve_from_r) — a rotating
        // visit's V_p J is 39 % of its flops; RLRA_SVD_VSOLVE=0 keeps V
        // accumulated.  A rejected solve re-runs the sweeps with V.
        static const bool vsolve_on = !std::getenv("RLRA_SVD_VSOLVE") || std::atoi(std::getenv("RLRA_SVD_VSOLVE")) != 0;
        bool skip_v = upper_tri && vsolve_on && m == n;
        for (int attempt = 0; attempt < 2; ++attempt) {
        if (attempt) {
            copy_mat(ctx, A, W);
            eye_mat(ctx, V);
            RLRA_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int) * 8, ctx.stream));
        }
        GramJacArgs g{};
        g.bar = ctx.gbar;
        g.W = W.m.p;
        g.ldw = W.m.ld;
        g.m = m;
        g.n = n;
        g.V = V.m.p;
        g.ldv = V.m.ld;
        g.nb = ceil_div(n, kSGB) + (ceil_div(n, kSGB) & 1);
        g.flags = flags.i();
        g.skip_v = skip_v ? 1 : 0;
        // W only: split every visit into two row-half tasks (RLRA_SGRAM_HALVES=0: one CTA per visit)
        static const bool halves_on = !std::getenv("RLRA_SGRAM_HALVES") || std::atoi(std::getenv("RLRA_SGRAM_HALVES")) != 0;
        g.halves = (skip_v && halves_on && ldw / kSCR >= 4) ? 1 : 0;
        const int snp = g.nb / 2;
        Buf xgb(ctx, g.halves ? sizeof(double) * size_t(4) * snp * kSXG : 8),
            xsb(ctx, g.halves ? sizeof(unsigned) * size_t(8) * snp : 8);
        if (g.halves) {
            RLRA_CUDA(cudaMemsetAsync(xsb.p, 0, sizeof(unsigned) * size_t(8) * snp, ctx.stream));
            g.xg = xgb.d();
            g.xstamp = static_cast<unsigned*>(xsb.p);
            g.xack = g.xstamp + 4 * snp;
        }
        static const bool sg_phases = std::getenv("RLRA_JACOBI_PHASES") != nullptr;
        Buf swb(ctx, sg_phases ? sizeof(long long) * (2 * kOneSidedSweepCap + 2) : 8);
        long long t_start = 0;
        if (sg_phases) {
            RLRA_CUDA(cudaMemsetAsync(swb.p, 0, sizeof(long long) * (2 * kOneSidedSweepCap + 2), ctx.stream));
            g.phase_clk = reinterpret_cast<long long*>(swb.p);
        }
        Buf verb(ctx, sizeof(unsigned) * 2 * g.nb);  // halves: one version per (half, block)
        RLRA_CUDA(cudaMemsetAsync(verb.p, 0, sizeof(unsigned) * 2 * g.nb, ctx.stream));
        g.ver = static_cast<unsigned*>(verb.p);
        const size_t nst = size_t(g.nb) + size_t(g.nb) * g.nb + g.nb / 2 + 2 * size_t(g.nb) + kOneSidedSweepCap;
        Buf stamps(ctx, sizeof(unsigned) * nst), cnt(ctx, sizeof(unsigned long long) * 4);
        RLRA_CUDA(cudaMemsetAsync(stamps.p, 0, sizeof(unsigned) * nst, ctx.stream));
        RLRA_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * 4, ctx.stream));
        g.mod = static_cast<unsigned*>(stamps.p);
        g.clean = g.mod + g.nb;
        g.vtick = g.clean + size_t(g.nb) * g.nb + g.nb / 2;
        g.vdone = g.vtick + g.nb;
        g.tasks = g.vdone + g.nb;
        g.counters = static_cast<unsigned long long*>(cnt.p);
        static unsigned* dbg_host = nullptr;
        if (std::getenv("RLRA_SGRAM_DEBUG")) {
            if (!dbg_host) RLRA_CUDA(cudaHostAlloc(&dbg_host, 4096, cudaHostAllocMapped));
            std::memset(dbg_host, 0, 4096);
            unsigned* dp = nullptr;
            RLRA_CUDA(cudaHostGetDevicePointer(&dp, dbg_host, 0));
            g.dbg = dp;
        }
        void* args[] = {&g};
        // visits are taken dynamically, so every SM can work (one CTA each):
        // CTAs beyond the np pair slots pick up the next round's ready pairs
        static const int sg_grid = std::getenv("RLRA_SGRAM_GRID") ? std::atoi(std::getenv("RLRA_SGRAM_GRID")) : 0;
        const int sgrid = sg_grid > 0 ? std::min(sg_grid, ctx.num_sms) : ctx.num_sms;
        RLRA_CUDA(cudaLaunchCooperativeKernel((void*)sgram_jacobi_kernel, dim3(sgrid), dim3(256), args, kSGramSmem,
                                              ctx.stream));
        if (g.dbg) {
            cudaError_t e = cudaErrorNotReady;
            for (int it = 0; it < 2000 && e == cudaErrorNotReady; ++it) {
                e = cudaStreamQuery(ctx.stream);
                if (e == cudaErrorNotReady) usleep(5000);
            }
            if (e == cudaErrorNotReady) {
                std::fprintf(stderr, "sgram debug: still running after 10 s; per-CTA (code task R):\n");
                for (int b = 0; b < sgrid; ++b)
                    std::fprintf(stderr, "%d:(%u %u %u) ", b, dbg_host[16 + 4 * b], dbg_host[17 + 4 * b], dbg_host[18 + 4 * b]);
                std::fprintf(stderr, "\n");
                if (g.halves) {
                    cudaStream_t s2;
                    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
                    std::vector<unsigned> hx(8 * snp), hv(2 * g.nb);
                    cudaMemcpyAsync(hx.data(), xsb.p, sizeof(unsigned) * hx.size(), cudaMemcpyDeviceToHost, s2);
                    cudaMemcpyAsync(hv.data(), verb.p, sizeof(unsigned) * hv.size(), cudaMemcpyDeviceToHost, s2);
                    cudaStreamSynchronize(s2);
                    std::fprintf(stderr, "xstamp/xack per slot (s: st0 st1 ack0 ack1):");
                    for (int q = 0; q < 2 * snp; ++q)
                        std::fprintf(stderr, " %d:(%u %u %u %u)", q, hx[2 * q], hx[2 * q + 1], hx[4 * snp + 2 * q], hx[4 * snp + 2 * q + 1]);
                    std::fprintf(stderr, "\nver half0/half1:");
                    for (int b = 0; b < g.nb; ++b) std::fprintf(stderr, " %d:(%u %u)", b, hv[b], hv[g.nb + b]);
                    std::fprintf(stderr, "\n");
                }
                std::fflush(stderr);
                std::abort();
            }
            std::fprintf(stderr, "sgram debug: %s; record %u code %u R %u half %u block %u cur %u want %u\n",
                         cudaGetErrorString(e), dbg_host[0], dbg_host[1], dbg_host[2], dbg_host[3], dbg_host[4],
                         dbg_host[5], dbg_host[6]);
        }
        if (std::getenv("RLRA_JACOBI_STATS")) {
            unsigned long long h[3];
            RLRA_CUDA(cudaMemcpyAsync(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
            RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
            std::fprintf(stderr, "sgram: %llu visits, %llu skipped (clean), %llu rotating%s%s\n", h[0], h[1], h[2],
                         skip_v ? " (W only)" : "", g.halves ? " (row halves)" : "");
        }
        if (sg_phases) {
            std::vector<long long> h(2 * kOneSidedSweepCap);
            RLRA_CUDA(cudaMemcpyAsync(h.data(), swb.p, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, ctx.stream));
            RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
            (void)t_start;
            std::fprintf(stderr, "sgram sweeps (end us, rotating visits):");
            for (int sw = 0; sw < kOneSidedSweepCap && h[2 * sw]; ++sw)
                std::fprintf(stderr, " [%d] %.0f %lld", sw, (h[2 * sw] - h[0]) * 1e-3, h[2 * sw + 1]);
            std::fprintf(stderr, "\n");
        }
        if (!skip_v) break;
        double defect = 0.0;
        const bool ok = vsolve_from_r(ctx, A, W.m, V.m, &defect);
        if (std::getenv("RLRA_JACOBI_STATS"))
            std::fprintf(stderr, "sgram: V = R^-1 W, max|V^T V - I| = %.3e (%s)\n", defect, ok ? "accepted" : "rejected");
        if (ok) break;
        skip_v = false;
        }
    } else if (forced != 4 && n > 2 * kGB) {
        // columns too long for shared memory: Gram block Jacobi (32-column blocks)
        static int gram_cap = 0;
        if (!gram_cap) {
            RLRA_CUDA(cudaFuncSetAttribute(gram_jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(kGramJacSmem)));
            int per = 0;
            RLRA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, gram_jacobi_kernel, 256, kGramJacSmem));
            gram_cap = std::max(1, per) * ctx.num_sms;
        }
        GramJacArgs g;
        g.bar = ctx.gbar;
        g.W = W.m.p;
        g.ldw = W.m.ld;
        g.m = m;
        g.n = n;
        g.V = V.m.p;
        g.ldv = V.m.ld;
        g.nb = ceil_div(n, kGB) + (ceil_div(n, kGB) & 1);
        g.flags = flags.i();
        g.inner_cap = kGInnerCap;
        g.phase_clk = nullptr;
        g.ver = nullptr;
        g.jbuf = nullptr;
        g.helpers = 0;
        void* args[] = {&g};
        const int grid = std::min(g.nb / 2, gram_cap);
        RLRA_CUDA(cudaLaunchCooperativeKernel((void*)gram_jacobi_kernel, dim3(grid), dim3(256), args, kGramJacSmem,
                                              ctx.stream));
    } else {
        const int pairs = (n + 1) / 2;
        const int G = coop_grid(ctx, (const void*)onesided_jacobi_kernel, ceil_div(pairs, kJacThreads / 32));
        a.bar = ctx.gbar;
        void* args[] = {&a};
        RLRA_CUDA(cudaLaunchCooperativeKernel((void*)onesided_jacobi_kernel, dim3(G), dim3(kJacThreads),
                                              args, 0, ctx.stream));
    }
    }
launched:
    ++ctx.launches;
    colnorm_kernel<<<ceil_div(n, 8), 256, 0, ctx.stream>>>(W.m.p, W.m.ld, m, n, sg.d());
    rank_desc_kernel<<<ceil_div(n, 256), 256, 0, ctx.stream>>>(sg.d(), n, rank.i());
    const int64_t tot = int64_t(std::max(m, n)) * n;
    svd_scatter_kernel<<<int(std::min<int64_t>((tot + 255) / 256, 4096)), 256, 0, ctx.stream>>>(
        W.m.p, W.m.ld, m, n, V.m.p, V.m.ld, n, sg.d(), rank.i(), U.p, U.ld, Vout.p, Vout.ld, sigma,
        needs.i());
    RLRA_LAUNCH_CHECK();
    ctx.launches += 3;
    if (prof.idx < 0 && ctx.svd_pending < 8) {
        // no host sync: the convergence status is checked when the API call
        // ends (the C-ABI guard), and the completion kernel runs always (it
        // leaves the columns alone when no singular value fell below the floor)
        const int slot = ctx.svd_pending++;
        ctx.svd_pending_mn[slot][0] = m;
        ctx.svd_pending_mn[slot][1] = n;
        RLRA_CUDA(cudaMemcpyAsync(ctx.h_flags + 32 + slot, flags.i() + 3, sizeof(int), cudaMemcpyDeviceToHost,
                                  ctx.stream));
        Buf done(ctx, sizeof(int) * n), r(ctx, sizeof(double) * m);
        completion_kernel<<<1, 256, 0, ctx.stream>>>(U.p, U.ld, m, n, needs.i(), done.i(), r.d());
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
        return;
    }
    RLRA_CUDA(cudaMemcpyAsync(ctx.h_flags, flags.p, sizeof(int) * 8, cudaMemcpyDeviceToHost,
                              ctx.stream));
    // any column needing completion?
    {
        // count needs on host: copy the n flags (small)
        std::vector<int> h(n);
        RLRA_CUDA(cudaMemcpyAsync(h.data(), needs.p, sizeof(int) * n, cudaMemcpyDeviceToHost,
                                  ctx.stream));
        RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
        if (ctx.h_flags[3] == RLRA_ECONV)
            raise(RLRA_ECONV, fmt("small_svd: no convergence after %d sweeps on %dx%d input",
                                  kOneSidedSweepCap, m, n));
        if (prof.idx >= 0) ctx.prof[prof.idx].K = ctx.h_flags[4];  // sweeps used
        bool any = false;
        for (int j = 0; j < n; ++j) any |= h[j] != 0;
        if (any) {
            Buf done(ctx, sizeof(int) * n), r(ctx, sizeof(double) * m);
            completion_kernel<<<1, 256, 0, ctx.stream>>>(U.p, U.ld, m, n, needs.i(), done.i(), r.d());
            RLRA_LAUNCH_CHECK();
            ++ctx.launches;
        }
    }
}

// the small_svd checks deferred in ctx (see Context::svd_pending)
void small_svd_deferred_checks(Context& ctx) {
    if (ctx.svd_pending == 0) return;
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    const int np = ctx.svd_pending;
    ctx.svd_pending = 0;
    for (int i = 0; i < np; ++i)
        if (ctx.h_flags[32 + i] == RLRA_ECONV)
            raise(RLRA_ECONV, fmt("small_svd: no convergence after %d sweeps on %dx%d input", kOneSidedSweepCap,
                                  ctx.svd_pending_mn[i][0], ctx.svd_pending_mn[i][1]));
}

void small_svd(Context& ctx, const DMat& A, const DMat& U, double* sigma, const DMat& V) {
    if (A.rows >= A.cols) return small_svd_tall(ctx, A, U, sigma, V);
    DMatBuf At(ctx, A.cols, A.rows);
    transpose_mat(ctx, A, At);
    small_svd_tall(ctx, At, V, sigma, U);
}

void sym_eig(Context& ctx, const DMat& T, double* values, const DMat& vectors) {
    const int n = int(T.rows);
    if (n == 0) return;
    // asymmetry guard (reference jacobi.hpp:76-84)
    double hv[2];
    Buf tn(ctx, sizeof(double)), part(ctx, sizeof(double) * 1024);
    sum_squares(ctx, T, tn.d());
    asym_kernel<<<64, 256, 0, ctx.stream>>>(T.p, T.ld, n, part.d());
    RLRA_LAUNCH_CHECK();
    ++ctx.launches;
    std::vector<double> pm(64);
    RLRA_CUDA(cudaMemcpyAsync(hv, tn.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    RLRA_CUDA(cudaMemcpyAsync(pm.data(), part.p, sizeof(double) * 64, cudaMemcpyDeviceToHost,
                              ctx.stream));
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    const double tnorm = sqrt(hv[0]);
    double asym = 0.0;
    for (double x : pm) asym = std::max(asym, x);
    if (tnorm > 0.0 && asym > 1e-12 * tnorm)
        raise(RLRA_ENUM, fmt("sym_eig: asymmetry %.3e exceeds 1e-12 relative to norm %.3e", asym,
                             tnorm));
    DMatBuf M(ctx, n, n), Uacc(ctx, n, n);
    copy_mat(ctx, T, M);
    eye_mat(ctx, Uacc);
    const int n2 = n + (n & 1);
    Buf cs(ctx, sizeof(double) * 3 * (n2 / 2 + 1)), status(ctx, sizeof(int)), d(ctx, sizeof(double) * n),
        rank(ctx, sizeof(int) * n);
    RLRA_CUDA(cudaMemsetAsync(status.p, 0, sizeof(int), ctx.stream));
    const int G = coop_grid(ctx, (const void*)twosided_jacobi_kernel,
                            std::max(1, std::min(ctx.num_sms, ceil_div(int64_t(n) * n, 4 * kJacThreads))));
    Buf part2(ctx, sizeof(double) * G);
    TwoSidedArgs a;
    a.M = M.m.p;
    a.ldm = M.m.ld;
    a.n = n;
    a.U = Uacc.m.p;
    a.ldu = Uacc.m.ld;
    a.cs = cs.d();
    a.part = part2.d();
    a.tnorm = tnorm;
    a.status = status.i();
    a.bar = ctx.gbar;
    void* args[] = {&a};
    RLRA_CUDA(cudaLaunchCooperativeKernel((void*)twosided_jacobi_kernel, dim3(G), dim3(kJacThreads),
                                          args, 0, ctx.stream));
    ++ctx.launches;
    diag_of_kernel<<<ceil_div(n, 256), 256, 0, ctx.stream>>>(M.m.p, M.m.ld, n, d.d());
    rank_desc_kernel<<<ceil_div(n, 256), 256, 0, ctx.stream>>>(d.d(), n, rank.i());
    eig_scatter_kernel<<<int(std::min<int64_t>((int64_t(n) * n + 255) / 256, 4096)), 256, 0,
                         ctx.stream>>>(d.d(), rank.i(), Uacc.m.p, Uacc.m.ld, n, values, vectors.p,
                                       vectors.ld);
    RLRA_LAUNCH_CHECK();
    ctx.launches += 3;
    RLRA_CUDA(cudaMemcpyAsync(ctx.h_flags, status.p, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
    RLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    if (ctx.h_flags[0] == RLRA_ECONV)
        raise(RLRA_ECONV, fmt("sym_eig: no convergence after %d sweeps (matrix norm %.3e)",
                              kTwoSidedSweepCap, tnorm));
}

}  // namespace rlra_b200
