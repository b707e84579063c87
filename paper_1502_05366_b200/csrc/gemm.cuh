// gemm.cuh — FP64 tensor-core GEMM for sm_100a (K1/K2/K7/K10 of SURVEY.md §2.2).
//
// Blackwell has no FP64 tcgen05/UMMA kind, so FP64 tensor math is
// mma.sync.m8n8k4.f64, which ptxas lowers to SASS DMMA.8x8x4 (measured peak
// 37.1 TFLOP/s on this pool's B200s, tools/fp64_peak.cu).  Operands are
// register-fed: global -> shared by a STAGES-deep cp.async pipeline (16-byte
// vectors when the leading dimension allows), shared -> registers with
// bank-conflict-free padded layouts, accumulators in registers.
//
// One kernel template serves every product on the path (reference
// core/matmul.hpp:68 with its four transpose cases):
//   NN  Y = A*Omega, Y = A*Z, U = Q*Vhat, Q_i*B_i        (matmul.hpp:20-29)
//   TN  Z = A^T*Y, Bt = A^T*Q, Gram Y^T*Y, Q^T*Q_i       (matmul.hpp:30-40)
//   NT  B*B^T (rsvd_v1)                                   (matmul.hpp:41-49)
// with three epilogues (plain store with alpha/beta, split-K partial store,
// and the fused residual "D = R - A*B, accumulate ||D||^2" used by the QB
// deflation and the CUR/verify residuals), an in-register Philox Omega B
// operand, a triangular-B K limit (Y*R^{-1}) and upper-tile-only mode (Gram).
#pragma once

#include "common.cuh"

namespace rlra_b200 {

enum GemmEpi { EPI_STORE = 0, EPI_SPLIT = 1, EPI_RESID = 2 };

struct GemmParams {
    int M, N, K;
    const double* A;
    int64_t lda;
    const double* B;
    int64_t ldb;
    double* C;
    int64_t ldc;
    double alpha, beta;
    int k_chunk;           // K extent per split (multiple of BK)
    int splits;
    int mt, nt;            // tile counts
    double* ws;            // EPI_SPLIT: slice s at ws + s*M*N, ld = M
    int tri_b_upper;       // B upper triangular: n-tile [n0,n1) only needs k < n1
    int upper_tiles_only;  // skip tiles with m-tile > n-tile (square C)
    // in-register Philox Omega (B operand, op N): element (k, n)
    uint64_t seed;
    int draw;
    int64_t krow0;
    // EPI_RESID: D = R - alpha*acc (stored to C when C != nullptr), sum D^2
    const double* R;
    int64_t ldr;
    double* partials;  // one per tile
    // tail-wave split (TMA path, EPI_STORE, splits == 1): CTAs from tail_base
    // on cover the last partial wave's tiles, each tile cut into tail_split
    // k-chunks of tail_kchunk whose partials go to tail_ws (reduced after)
    int tail_base;     // first tail CTA (INT_MAX: none)
    int tail_split;
    int tail_kchunk;
    double* tail_ws;   // [tail tile][part][128 x 128]
};

// ---------------------------------------------------------------- philox ---
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k.x += 0x9E3779B9u;
            k.y += 0xBB67AE85u;
        }
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}

// Exact float -> double widening with integer ops only (sign, exponent
// re-bias, mantissa shift): bit-identical to double(f) for normal floats and
// zero, and keeps the conversion off the FP64 pipe the DMMA sketch saturates.
// (Box-Muller outputs are never subnormal, infinite or NaN.)
__device__ __forceinline__ double f32_to_f64_bits(float f) {
    const uint32_t u = __float_as_uint(f);
    const uint32_t e = (u >> 23) & 0xffu;
    const uint32_t hi = e ? ((u & 0x80000000u) | ((e + 896u) << 20) | ((u & 0x7fffffu) >> 3)) : (u & 0x80000000u);
    const uint32_t lo = e ? (u << 29) : 0u;
    return __hiloint2double(int(hi), int(lo));
}

// Four N(0,1) deviates for rows 4*(k>>2)+{0..3} of column n in draw `draw`.
// Box-Muller in fp32 on the FP32/SFU pipes (the FP64 pipe is the bottleneck);
// the deviates only need to be Gaussian, the product with them is exact FP64.
__device__ __forceinline__ void philox_normal4(uint64_t seed, int draw, int64_t k, int64_t n,
                                               double out[4]) {
    const uint4 ctr = make_uint4(uint32_t(uint64_t(k) >> 2), uint32_t(n), uint32_t(draw),
                                 uint32_t(uint64_t(k) >> 34));
    const uint4 x = philox4x32_10(ctr, make_uint2(uint32_t(seed), uint32_t(seed >> 32)));
    const float s24 = 5.9604644775390625e-8f;  // 2^-24
    const float u1a = float((x.x >> 8) + 1u) * s24;  // (0,1]
    const float u2a = float(x.y >> 8) * s24;         // [0,1)
    const float u1b = float((x.z >> 8) + 1u) * s24;
    const float u2b = float(x.w >> 8) * s24;
    const float ra = sqrtf(-2.0f * __logf(u1a));
    const float rb = sqrtf(-2.0f * __logf(u1b));
    float sa, ca, sb, cb;
    __sincosf(6.283185307179586f * u2a, &sa, &ca);
    __sincosf(6.283185307179586f * u2b, &sb, &cb);
    out[0] = f32_to_f64_bits(ra * ca);
    out[1] = f32_to_f64_bits(ra * sa);
    out[2] = f32_to_f64_bits(rb * cb);
    out[3] = f32_to_f64_bits(rb * sb);
}

// ------------------------------------------------------------- cp.async ---
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Shared-memory tile geometry.  "KM" (k-major) tiles are [BK][X+4]: used when
// the operand is contiguous along its M/N index in global memory.  "XM" tiles
// are [X][BK+4]: operand contiguous along k.  Both paddings make the m8n8k4
// fragment loads (8 x-values by 4 k-values per warp) conflict-free per
// half-warp, and keep rows 16-byte aligned for cp.async.16.
template <bool KM, int X, int BK>
struct TileGeo {
    static constexpr int pitch = KM ? (X + 4) : (BK + 4);
    static constexpr int elems = KM ? BK * (X + 4) : X * (BK + 4);
    __device__ static __forceinline__ int off(int k, int x) { return KM ? k * pitch + x : x * pitch + k; }
};

// Load a BK x X tile of op(M) starting at (k0, x0) into smem.
//   KM: element (k, x) at g[x + k*ld]   (x contiguous)
//   XM: element (k, x) at g[k + x*ld]   (k contiguous)
// Elements with k >= kmax or x >= xmax are zero-filled.
template <bool KM, int X, int BK, int NT, bool VEC>
__device__ __forceinline__ void load_tile(double* s, const double* g, int64_t ld, int x0, int k0,
                                          int xmax, int kmax) {
    using G = TileGeo<KM, X, BK>;
    constexpr int W = VEC ? 2 : 1;  // doubles per copy
    constexpr int CONTIG = KM ? X : BK;
    constexpr int OTHER = KM ? BK : X;
    constexpr int CHUNKS = (CONTIG / W) * OTHER;
    static_assert(CHUNKS % NT == 0, "tile/thread mismatch");
#pragma unroll
    for (int it = 0; it < CHUNKS / NT; ++it) {
        const int c = it * NT + threadIdx.x;
        const int o = c / (CONTIG / W);
        const int ci = (c % (CONTIG / W)) * W;
        int k, x, rem;
        if (KM) {
            k = k0 + o;
            x = x0 + ci;
            rem = (k < kmax) ? (xmax - x) : 0;
        } else {
            x = x0 + o;
            k = k0 + ci;
            rem = (x < xmax) ? (kmax - k) : 0;
        }
        rem = rem < 0 ? 0 : (rem > W ? W : rem);
        double* dst = s + (KM ? G::off(o, ci) : G::off(ci, o));
        const double* src = rem > 0 ? g + (KM ? (int64_t(x) + int64_t(k) * ld) : (int64_t(k) + int64_t(x) * ld)) : g;
        if (VEC)
            cp_async16(dst, src, rem * 8);
        else
            cp_async8(dst, src, rem * 8);
    }
}

// Philox Omega tile: B is (K x N) "XM" layout [n][k]; generated, not loaded.
template <int BN, int BK, int NT>
__device__ __forceinline__ void gen_omega_tile(double* s, const GemmParams& p, int n0, int k0, int kmax) {
    using G = TileGeo<false, BN, BK>;
    constexpr int GROUPS = BN * (BK / 4);
    static_assert(GROUPS % NT == 0, "omega tile/thread mismatch");
#pragma unroll
    for (int it = 0; it < GROUPS / NT; ++it) {
        const int g = it * NT + threadIdx.x;
        const int nl = g / (BK / 4);
        const int kl = (g % (BK / 4)) * 4;
        const int n = n0 + nl, k = k0 + kl;
        double v[4] = {0.0, 0.0, 0.0, 0.0};
        if (n < p.N && k < kmax) {
            philox_normal4(p.seed, p.draw, p.krow0 + k, n, v);
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (k + t >= kmax) v[t] = 0.0;
        }
        double* dst = s + G::off(kl, nl);
        *reinterpret_cast<double2*>(dst) = make_double2(v[0], v[1]);
        *reinterpret_cast<double2*>(dst + 2) = make_double2(v[2], v[3]);
    }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool A_KM, bool B_KM, bool VEC,
          int EPI, bool PHILOX>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32, 1) dgemm_kernel(const GemmParams p) {
    constexpr int NWM = BM / WM, NWN = BN / WN;
    constexpr int NT = NWM * NWN * 32;
    constexpr int MF = WM / 8, NF = WN / 8;
    using GA = TileGeo<A_KM, BM, BK>;
    using GB = TileGeo<B_KM, BN, BK>;
    extern __shared__ __align__(16) double smem[];
    double* sA = smem;
    double* sB = smem + STAGES * GA::elems;

    const int tile = blockIdx.x;
    const int nt_i = tile % p.nt;
    const int rest = tile / p.nt;
    const int mt_i = rest % p.mt;
    const int split = rest / p.mt;
    if (p.upper_tiles_only && mt_i > nt_i) return;
    const int m0 = mt_i * BM, n0 = nt_i * BN;
    const int k_begin = split * p.k_chunk;
    int k_end = min(p.K, k_begin + p.k_chunk);
    if (p.tri_b_upper) k_end = min(k_end, n0 + BN);
    const int nk = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp % NWM, wn = warp / NWM;
    const int lr = lane >> 2, lc = lane & 3;

    double acc[MF][NF][2];
#pragma unroll
    for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    auto issue = [&](int kt) {
        const int st = kt % STAGES;
        const int k0 = k_begin + kt * BK;
        load_tile<A_KM, BM, BK, NT, VEC>(sA + st * GA::elems, p.A, p.lda, m0, k0, p.M, k_end);
        if (PHILOX)
            gen_omega_tile<BN, BK, NT>(sB + st * GB::elems, p, n0, k0, k_end);
        else
            load_tile<B_KM, BN, BK, NT, VEC>(sB + st * GB::elems, p.B, p.ldb, n0, k0, p.N, k_end);
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) issue(s);
        cp_async_commit();
    }

    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        if (kt + STAGES - 1 < nk) issue(kt + STAGES - 1);
        cp_async_commit();
        const double* a_s = sA + (kt % STAGES) * GA::elems;
        const double* b_s = sB + (kt % STAGES) * GB::elems;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[MF], bf[NF];
#pragma unroll
            for (int i = 0; i < MF; ++i) af[i] = a_s[GA::off(kk + lc, wm * WM + i * 8 + lr)];
#pragma unroll
            for (int j = 0; j < NF; ++j) bf[j] = b_s[GB::off(kk + lc, wn * WN + j * 8 + lr)];
#pragma unroll
            for (int i = 0; i < MF; ++i)
#pragma unroll
                for (int j = 0; j < NF; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    cp_async_wait<0>();

    // ---------------------------------------------------------- epilogue ---
    double local = 0.0;
#pragma unroll
    for (int i = 0; i < MF; ++i) {
        const int row = m0 + wm * WM + i * 8 + lr;
        // EPI_RESID: this fragment row's R values first (C may alias R, so
        // loads inside the store loop would each wait a round trip)
        double rin[NF][2];
        if (EPI == EPI_RESID) {
#pragma unroll
            for (int j = 0; j < NF; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int col = n0 + wn * WN + j * 8 + lc * 2 + h;
                    rin[j][h] = (row < p.M && col < p.N) ? p.R[row + int64_t(col) * p.ldr] : 0.0;
                }
        }
#pragma unroll
        for (int j = 0; j < NF; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = n0 + wn * WN + j * 8 + lc * 2 + h;
                if (row < p.M && col < p.N) {
                    const double v = acc[i][j][h];
                    if (EPI == EPI_STORE) {
                        double* c = p.C + row + int64_t(col) * p.ldc;
                        *c = p.beta == 0.0 ? p.alpha * v : p.alpha * v + p.beta * *c;
                    } else if (EPI == EPI_SPLIT) {
                        p.ws[int64_t(split) * p.M * p.N + row + int64_t(col) * p.M] = v;
                    } else {
                        const double d = rin[j][h] - p.alpha * v;
                        if (p.C) p.C[row + int64_t(col) * p.ldc] = d;
                        local += d * d;
                    }
                }
            }
        }
    }
    if (EPI == EPI_RESID) {
        // fixed-order block reduction: warp tree, then warp 0 over warps
        __shared__ double red[NT / 32];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
        __syncthreads();
        if (lane == 0) red[warp] = local;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < NT / 32; ++w) t += red[w];
            p.partials[tile] = t;
        }
    }
}

// --------------------------------------------- warp-specialized variant ---
// Same tiles, fragments and epilogues as dgemm_kernel, but the CTA is split
// into a producer warpgroup (cp.async for A and B, or in-register Philox for
// Omega) and 2 consumer warpgroups (DMMA).  Stages are handed over through
// mbarriers (full: producer -> consumers, empty: consumers -> producer), so
// consumer warps never wait on each other and the Philox generation runs
// concurrently with the tensor pipe instead of at the stage boundary.
// setmaxnreg moves registers from the producer (56) to the consumers (224).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t* b) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool A_KM, bool B_KM, bool VEC,
          int EPI, bool PHILOX>
__global__ void __launch_bounds__(128 + (BM / WM) * (BN / WN) * 32, 1) dgemm_ws_kernel(const GemmParams p) {
    constexpr int NWM = BM / WM, NWN = BN / WN;
    constexpr int NCW = NWM * NWN;  // consumer warps
    constexpr int MF = WM / 8, NF = WN / 8;
    using GA = TileGeo<A_KM, BM, BK>;
    using GB = TileGeo<B_KM, BN, BK>;
    extern __shared__ __align__(16) double smem[];
    double* sA = smem;
    double* sB = smem + STAGES * GA::elems;
    __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
    __shared__ double red[NCW];

    const int tile = blockIdx.x;
    const int nt_i = tile % p.nt;
    const int rest = tile / p.nt;
    const int mt_i = rest % p.mt;
    const int split = rest / p.mt;
    if (p.upper_tiles_only && mt_i > nt_i) return;
    const int m0 = mt_i * BM, n0 = nt_i * BN;
    const int k_begin = split * p.k_chunk;
    int k_end = min(p.K, k_begin + p.k_chunk);
    if (p.tri_b_upper) k_end = min(k_end, n0 + BN);
    const int nk = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], PHILOX ? 256u : 128u);
            mbar_init(&empty_bar[s], unsigned(NCW));
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (threadIdx.x < 128) {
        // ------------------------------------------------------ producer ---
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n");
        for (int kt = 0; kt < nk; ++kt) {
            const int st = kt % STAGES;
            if (kt >= STAGES) mbar_wait(&empty_bar[st], ((kt / STAGES) - 1) & 1);
            const int k0 = k_begin + kt * BK;
            load_tile<A_KM, BM, BK, 128, VEC>(sA + st * GA::elems, p.A, p.lda, m0, k0, p.M, k_end);
            if (PHILOX) {
                gen_omega_tile<BN, BK, 128>(sB + st * GB::elems, p, n0, k0, k_end);
                mbar_arrive(&full_bar[st]);
            } else {
                load_tile<B_KM, BN, BK, 128, VEC>(sB + st * GB::elems, p.B, p.ldb, n0, k0, p.N, k_end);
            }
            mbar_arrive_cp_async(&full_bar[st]);
        }
        return;
    }
    // -------------------------------------------------------- consumers ---
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n");
    const int warp = (threadIdx.x >> 5) - 4, lane = threadIdx.x & 31;
    const int wm = warp % NWM, wn = warp / NWM;
    const int lr = lane >> 2, lc = lane & 3;
    double acc[MF][NF][2];
#pragma unroll
    for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < nk; ++kt) {
        const int st = kt % STAGES;
        mbar_wait(&full_bar[st], (kt / STAGES) & 1);
        const double* a_s = sA + st * GA::elems;
        const double* b_s = sB + st * GB::elems;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[MF], bf[NF];
#pragma unroll
            for (int i = 0; i < MF; ++i) af[i] = a_s[GA::off(kk + lc, wm * WM + i * 8 + lr)];
#pragma unroll
            for (int j = 0; j < NF; ++j) bf[j] = b_s[GB::off(kk + lc, wn * WN + j * 8 + lr)];
#pragma unroll
            for (int i = 0; i < MF; ++i)
#pragma unroll
                for (int j = 0; j < NF; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[st]);
    }

    double local = 0.0;
#pragma unroll
    for (int i = 0; i < MF; ++i) {
        const int row = m0 + wm * WM + i * 8 + lr;
        // EPI_RESID: this fragment row's R values first (C may alias R, so
        // loads inside the store loop would each wait a round trip)
        double rin[NF][2];
        if (EPI == EPI_RESID) {
#pragma unroll
            for (int j = 0; j < NF; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int col = n0 + wn * WN + j * 8 + lc * 2 + h;
                    rin[j][h] = (row < p.M && col < p.N) ? p.R[row + int64_t(col) * p.ldr] : 0.0;
                }
        }
#pragma unroll
        for (int j = 0; j < NF; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = n0 + wn * WN + j * 8 + lc * 2 + h;
                if (row < p.M && col < p.N) {
                    const double v = acc[i][j][h];
                    if (EPI == EPI_STORE) {
                        double* c = p.C + row + int64_t(col) * p.ldc;
                        *c = p.beta == 0.0 ? p.alpha * v : p.alpha * v + p.beta * *c;
                    } else if (EPI == EPI_SPLIT) {
                        p.ws[int64_t(split) * p.M * p.N + row + int64_t(col) * p.M] = v;
                    } else {
                        const double d = rin[j][h] - p.alpha * v;
                        if (p.C) p.C[row + int64_t(col) * p.ldc] = d;
                        local += d * d;
                    }
                }
            }
        }
    }
    if (EPI == EPI_RESID) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
        if (lane == 0) red[warp] = local;
        asm volatile("bar.sync 1, %0;\n" ::"n"(NCW * 32));
        if (warp == 0 && lane == 0) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < NCW; ++w) t += red[w];
            p.partials[tile] = t;
        }
    }
}

// ------------------------------------------------------------ host side ---
enum class Op { N = 0, T = 1 };

struct GemmOpts {
    int epi = EPI_STORE;
    bool tri_b_upper = false;
    bool upper_tiles_only = false;
    bool philox_b = false;
    uint64_t seed = 0;
    int draw = 0;
    int64_t krow0 = 0;
    const double* R = nullptr;  // EPI_RESID
    int64_t ldr = 0;
    double* resid_sq = nullptr;  // EPI_RESID: device scalar receiving sum D^2
    int force_splits = 0;
};

// Materialise the Philox Omega the sketch GEMM generates in-register:
// out(i, j) = philox_normal(seed, draw, row0 + i, j), bit-identical to the
// values gen_omega_tile feeds the DMMA pipe.
void philox_fill(Context& ctx, const DMat& out, uint64_t seed, int draw, int64_t row0);

// C (M x N) = alpha * op(A) * op(B) + beta * C on ctx.stream.
void gemm(Context& ctx, Op opa, Op opb, int M, int N, int K, double alpha, const double* A,
          int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
          const GemmOpts& o = GemmOpts());

inline void gemm(Context& ctx, Op opa, Op opb, double alpha, const DMat& A, const DMat& B,
                 double beta, const DMat& C, const GemmOpts& o = GemmOpts()) {
    const int M = int(opa == Op::N ? A.rows : A.cols);
    const int K = int(opa == Op::N ? A.cols : A.rows);
    const int N = int(opb == Op::N ? B.cols : B.rows);
    gemm(ctx, opa, opb, M, N, K, alpha, A.p, A.ld, B.p, B.ld, beta, C.p, C.ld, o);
}

}  // namespace rlra_b200
