// gemm.cu — launcher for the FP64 DMMA GEMM family (see gemm.cuh).
#include <climits>
#include <cstdlib>
#include <string>

#include <cudaTypedefs.h>

#include "gemm.cuh"
#include "gemm_tma.cuh"
#include "reduce.cuh"

namespace rlra_b200 {

namespace {

// 128x128 CTA tile, 8 warps of 64x32 (2 warps per scheduler)
struct CfgBig {
    static constexpr int BM = 128, BN = 128, BK = 16, WM = 64, WN = 32, STAGES = 4;
    static constexpr bool WS = true;
};
// 128x128 CTA tile, 16 warps of 32x32 (4 warps per scheduler: more DMMA
// issue candidates per SMSP at the same shared-memory tile)
struct CfgBig16 {
    static constexpr int BM = 128, BN = 128, BK = 16, WM = 32, WN = 32, STAGES = 4;
    static constexpr bool WS = false;
};

int big_cfg_choice() {
    static int choice = [] {
        const char* e = std::getenv("RLRA_GEMM_CFG");
        if (e && std::string(e) == "w8") return 8;
        if (e && std::string(e) == "w16") return 16;
        return 8;
    }();
    return choice;
}
struct CfgSmall {
    static constexpr int BM = 64, BN = 64, BK = 16, WM = 32, WN = 32, STAGES = 4;
    static constexpr bool WS = false;
};

template <class Cfg, bool A_KM, bool B_KM>
constexpr size_t smem_bytes() {
    return sizeof(double) * Cfg::STAGES *
           (TileGeo<A_KM, Cfg::BM, Cfg::BK>::elems + TileGeo<B_KM, Cfg::BN, Cfg::BK>::elems);
}

bool ws_choice() {
    static bool ws = [] {
        const char* e = std::getenv("RLRA_GEMM_WS");
        return !(e && std::string(e) == "0");
    }();
    return ws;
}

template <class Cfg, bool A_KM, bool B_KM, bool VEC, int EPI, bool PHILOX>
void launch_cfg(Context& ctx, const GemmParams& p) {
    constexpr size_t smem = smem_bytes<Cfg, A_KM, B_KM>();
    const int64_t grid = int64_t(p.mt) * p.nt * p.splits;
    constexpr int consumers = (Cfg::BM / Cfg::WM) * (Cfg::BN / Cfg::WN) * 32;
    bool launched = false;
    if constexpr (Cfg::WS) {
      if (ws_choice()) {
        auto kern = dgemm_ws_kernel<Cfg::BM, Cfg::BN, Cfg::BK, Cfg::WM, Cfg::WN, Cfg::STAGES, A_KM, B_KM,
                                    VEC, EPI, PHILOX>;
        static bool attr_set = false;  // per instantiation
        if (!attr_set) {
            RLRA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            attr_set = true;
        }
        kern<<<dim3(unsigned(grid)), 128 + consumers, smem, ctx.stream>>>(p);
        launched = true;
      }
    }
    if (!launched) {
        auto kern = dgemm_kernel<Cfg::BM, Cfg::BN, Cfg::BK, Cfg::WM, Cfg::WN, Cfg::STAGES, A_KM, B_KM, VEC,
                                 EPI, PHILOX>;
        static bool attr_set = false;  // per instantiation
        if (!attr_set) {
            RLRA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            attr_set = true;
        }
        kern<<<dim3(unsigned(grid)), consumers, smem, ctx.stream>>>(p);
    }
    RLRA_LAUNCH_CHECK();
    ++ctx.launches;
}

template <class Cfg, bool A_KM, bool B_KM, bool VEC>
void launch_epi(Context& ctx, const GemmParams& p, int epi, bool philox) {
    if (philox) {
        if constexpr (!B_KM) {
            if (epi == EPI_STORE) return launch_cfg<Cfg, A_KM, B_KM, VEC, EPI_STORE, true>(ctx, p);
            if (epi == EPI_SPLIT) return launch_cfg<Cfg, A_KM, B_KM, VEC, EPI_SPLIT, true>(ctx, p);
        }
        raise(RLRA_EINVAL, "gemm: Philox B operand needs op(B)=N and a store/split epilogue");
    }
    if (epi == EPI_STORE) return launch_cfg<Cfg, A_KM, B_KM, VEC, EPI_STORE, false>(ctx, p);
    if (epi == EPI_SPLIT) return launch_cfg<Cfg, A_KM, B_KM, VEC, EPI_SPLIT, false>(ctx, p);
    return launch_cfg<Cfg, A_KM, B_KM, VEC, EPI_RESID, false>(ctx, p);
}

template <class Cfg>
void launch_ops(Context& ctx, Op opa, Op opb, bool vec, const GemmParams& p, int epi, bool philox) {
    const bool akm = opa == Op::N, bkm = opb == Op::T;
#define RLRA_DISPATCH(AK, BK_)                                                   \
    if (akm == AK && bkm == BK_) {                                               \
        if (vec) return launch_epi<Cfg, AK, BK_, true>(ctx, p, epi, philox);     \
        return launch_epi<Cfg, AK, BK_, false>(ctx, p, epi, philox);             \
    }
    RLRA_DISPATCH(true, false)
    RLRA_DISPATCH(false, false)
    RLRA_DISPATCH(true, true)
    RLRA_DISPATCH(false, true)
#undef RLRA_DISPATCH
}

// ------------------------------------------------------------- TMA path ---
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

bool tail_choice() {
    static bool on = [] {
        const char* e = std::getenv("RLRA_GEMM_TAIL");
        return !(e && std::string(e) == "0");
    }();
    return on;
}

bool tma_choice() {
    static bool on = [] {
        const char* e = std::getenv("RLRA_GEMM_TMA");
        return !(e && std::string(e) == "0");
    }();
    return on;
}

// 2-D FP64 tensor map over a column-major matrix: dim0 contiguous (d0
// elements), dim1 strided by ld; 128-byte swizzled boxes of b0 x b1.
void encode_map(CUtensorMap* m, const double* base, int64_t d0, int64_t d1, int64_t ld, int b0, int b1) {
    auto enc = tensor_map_encoder();
    if (!enc) raise(RLRA_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    const cuuint64_t dims[2] = {cuuint64_t(d0), cuuint64_t(d1)};
    const cuuint64_t strides[1] = {cuuint64_t(ld) * 8};
    const cuuint32_t box[2] = {cuuint32_t(b0), cuuint32_t(b1)};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) raise(RLRA_ECUDA, fmt("cuTensorMapEncodeTiled failed (%d)", int(r)));
}

// x-contiguous A (M x K, M % 16 == 0) as the 3-D tensor (16, K, M/16): a
// (16, BK, 8) box is a 128 x BK slice in the eight-box swizzled layout.
void encode_map3_km(CUtensorMap* m, const double* base, int64_t M, int64_t K, int64_t ld) {
    auto enc = tensor_map_encoder();
    if (!enc) raise(RLRA_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    const cuuint64_t dims[3] = {16, cuuint64_t(K), cuuint64_t(M / 16)};
    const cuuint64_t strides[2] = {cuuint64_t(ld) * 8, 128};
    const cuuint32_t box[3] = {16, cuuint32_t(kTBK), cuuint32_t(kTBM / 16)};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) raise(RLRA_ECUDA, fmt("cuTensorMapEncodeTiled (3-D) failed (%d)", int(r)));
}

template <bool A_KM, int EPI, bool PHILOX, int CL>
void launch_tma_cfg(Context& ctx, const GemmParams& p, const TmaPair& maps) {
    auto kern = dgemm_tma_kernel<A_KM, EPI, PHILOX, CL>;
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        RLRA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTmaSmem)));
        attr_set = true;
    }
    if (CL == 1) {
        int64_t grid = int64_t(p.mt) * p.nt * p.splits;
        if (p.tail_base != INT_MAX) grid = p.tail_base + (grid - p.tail_base) * p.tail_split;
        kern<<<dim3(unsigned(grid)), 384, kTmaSmem, ctx.stream>>>(p, maps);
    } else {
        const int64_t grid = int64_t(ceil_div(p.mt, CL)) * CL * p.nt * p.splits;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(grid));
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = kTmaSmem;
        cfg.stream = ctx.stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CL;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        RLRA_CUDA(cudaLaunchKernelEx(&cfg, kern, p, maps));
    }
    RLRA_LAUNCH_CHECK();
    ++ctx.launches;
}

int omega_cluster_choice() {
    static int cl = [] {
        const char* e = std::getenv("RLRA_OMEGA_CLUSTER");
        // pairs: 4-CTA clusters strand SMs of the 18-19-SM GPCs at 1 CTA/SM
        return e ? std::atoi(e) : 2;
    }();
    return cl;
}

template <bool A_KM>
void launch_tma_epi(Context& ctx, const GemmParams& p, const TmaPair& maps, int epi, bool philox) {
    if (philox) {
        // >= 4 m-tiles: cluster pairs of m-tiles share each generated Omega slice
        const int cl = p.mt >= 4 ? omega_cluster_choice() : 1;
        if (epi == EPI_STORE)
            return cl == 4 ? launch_tma_cfg<A_KM, EPI_STORE, true, 4>(ctx, p, maps)
                 : cl == 2 ? launch_tma_cfg<A_KM, EPI_STORE, true, 2>(ctx, p, maps)
                           : launch_tma_cfg<A_KM, EPI_STORE, true, 1>(ctx, p, maps);
        if (epi == EPI_SPLIT)
            return cl == 4 ? launch_tma_cfg<A_KM, EPI_SPLIT, true, 4>(ctx, p, maps)
                 : cl == 2 ? launch_tma_cfg<A_KM, EPI_SPLIT, true, 2>(ctx, p, maps)
                           : launch_tma_cfg<A_KM, EPI_SPLIT, true, 1>(ctx, p, maps);
        raise(RLRA_EINVAL, "gemm: Philox B operand needs a store/split epilogue");
    }
    if (epi == EPI_STORE) return launch_tma_cfg<A_KM, EPI_STORE, false, 1>(ctx, p, maps);
    if (epi == EPI_SPLIT) return launch_tma_cfg<A_KM, EPI_SPLIT, false, 1>(ctx, p, maps);
    return launch_tma_cfg<A_KM, EPI_RESID, false, 1>(ctx, p, maps);
}

// C tile = alpha * sum of the tail parts + beta * C, for the tail tiles
__global__ void tail_reduce_kernel(const double* ws, int split, int tail_base, int ntail, int mt, int nt, int M,
                                   int N, double alpha, double beta, double* C, int64_t ldc) {
    const int64_t per = int64_t(kTBM) * kTBN;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(ntail) * per;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int t = int(e / per), li = int(e % per);
        const int tile = tail_base + t;
        const int row = (tile / nt) % mt * kTBM + li % kTBM, col = tile % nt * kTBN + li / kTBM;
        if (row >= M || col >= N) continue;
        double s = 0.0;
        for (int q = 0; q < split; ++q) s += ws[(int64_t(t) * split + q) * per + li];
        double* c = C + row + int64_t(col) * ldc;
        *c = beta == 0.0 ? alpha * s : alpha * s + beta * *c;
    }
}

__global__ void split_reduce_kernel(const double* ws, int splits, int M, int N, double alpha,
                                    double beta, double* C, int64_t ldc, int upper_tile, int tile) {
    const int64_t total = int64_t(M) * N;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int row = int(e % M);
        const int col = int(e / M);
        if (upper_tile && row / tile > col / tile) continue;
        double s = 0.0;
        for (int t = 0; t < splits; ++t) s += ws[int64_t(t) * total + e];
        double* c = C + row + int64_t(col) * ldc;
        *c = beta == 0.0 ? alpha * s : alpha * s + beta * *c;
    }
}

__global__ void philox_fill_kernel(double* out, int64_t ld, int64_t rows, int64_t cols, uint64_t seed,
                                   int draw, int64_t row0) {
    // one thread per group of 4 consecutive global rows of one column
    const int64_t g0 = row0 >> 2, g1 = (row0 + rows + 3) >> 2;
    const int64_t groups = (g1 - g0) * cols;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < groups;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t j = e / (g1 - g0), g = g0 + e % (g1 - g0);
        double v[4];
        philox_normal4(seed, draw, g * 4, j, v);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int64_t r = g * 4 + t - row0;
            if (r >= 0 && r < rows) out[r + j * ld] = v[t];
        }
    }
}

}  // namespace

void philox_fill(Context& ctx, const DMat& out, uint64_t seed, int draw, int64_t row0) {
    if (out.rows <= 0 || out.cols <= 0) return;
    const int64_t groups = ((out.rows + 7) / 4) * out.cols;
    const int blocks = int(std::min<int64_t>((groups + 255) / 256, int64_t(ctx.num_sms) * 16));
    philox_fill_kernel<<<blocks, 256, 0, ctx.stream>>>(out.p, out.ld, out.rows, out.cols, seed, draw,
                                                       row0);
    RLRA_LAUNCH_CHECK();
    ++ctx.launches;
}

void gemm(Context& ctx, Op opa, Op opb, int M, int N, int K, double alpha, const double* A,
          int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
          const GemmOpts& o) {
    if (M <= 0 || N <= 0) return;
    if (K <= 0 && o.epi == EPI_STORE) {
        // C = beta*C (alpha*0): reuse the split reducer with zero splits
        split_reduce_kernel<<<ctx.num_sms * 4, 256, 0, ctx.stream>>>(nullptr, 0, M, N, alpha, beta,
                                                                      C, ldc, 0, 1);
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
        return;
    }
    // 128 x 128 tiles unless they leave most SMs idle with little k to split:
    // an l x l Gram (<= 4 big tiles) or a short-k product (k <= 1024) of
    // fewer than 100 big tiles runs on 64 x 64 tiles, up to three CTAs per SM
    // (C1: the k = 210 products 40 -> 20 us, its Grams 32 -> 24 us; the
    // long-k sketch products stay faster on big tiles).
    // RLRA_GEMM_BIG_MIN_TILES=t replaces the rule by "big iff >= t tiles".
    static const int big_min_tiles = [] {
        const char* e = std::getenv("RLRA_GEMM_BIG_MIN_TILES");
        return e ? std::atoi(e) : -1;
    }();
    const int64_t big_tiles = int64_t(ceil_div(M, CfgBig::BM)) * ceil_div(N, CfgBig::BN);
    // (also k <= 128 at any size — the QB deflation W -= Q_i B_i, b = 100: its
    // epilogue streams R and D once per tile, and three CTAs per SM overlap
    // one tile's epilogue with the next tiles' k-loops: C2 41.5 -> 37.4 ms)
    const bool few = big_min_tiles >= 0 ? big_tiles < big_min_tiles
                                        : (big_tiles <= 4 || (big_tiles < 100 && K <= 1024) || K <= 128);
    const bool big = M >= 96 && N >= 96 && !few;
    const int BM = big ? CfgBig::BM : CfgSmall::BM;
    const int BN = big ? CfgBig::BN : CfgSmall::BN;
    const int BK = 16;
    const int per_sm = big ? 1 : 3;

    GemmParams p{};
    p.M = M;
    p.N = N;
    p.K = K;
    p.A = A;
    p.lda = lda;
    p.B = B;
    p.ldb = ldb;
    p.C = C;
    p.ldc = ldc;
    p.alpha = alpha;
    p.beta = beta;
    p.mt = ceil_div(M, BM);
    p.nt = ceil_div(N, BN);
    p.tri_b_upper = o.tri_b_upper;
    p.upper_tiles_only = o.upper_tiles_only;
    p.seed = o.seed;
    p.draw = o.draw;
    p.krow0 = o.krow0;
    p.R = o.R;
    p.ldr = o.ldr;
    p.tail_base = INT_MAX;
    p.tail_split = 1;

    int64_t tiles = int64_t(p.mt) * p.nt;
    if (o.upper_tiles_only) tiles = int64_t(p.mt) * (p.mt + 1) / 2;
    const int64_t cap = int64_t(ctx.num_sms) * per_sm;
    // split-K where it pays against wave quantization.  Cost model per split
    // count s: (CTA waves) x (one CTA's k-chunk at the DMMA rate) + the
    // deterministic reduction ((s+1) M N doubles through HBM) + one launch.
    int splits = 1;
    if (o.epi != EPI_RESID && !o.tri_b_upper) {
        static const int env_splits = std::getenv("RLRA_GEMM_SPLITS") ? std::atoi(std::getenv("RLRA_GEMM_SPLITS")) : 0;
        if (o.force_splits > 0 || env_splits > 0) {
            splits = o.force_splits > 0 ? o.force_splits : env_splits;
        } else {
            const double cta_rate = 2.5e11 / per_sm;  // FP64 flop/s of one CTA (37 TF / 148 SMs)
            const double hbm = 5.0e12;                // B/s, reduction traffic
            // without split-K the TMA path splits the last partial wave's tiles
            // into s_t k-chunks (tail split, below): that wave then costs
            // 1/s_t of a tile plus a small reduction, not a whole tile
            const bool vec_ok = (lda % 2 == 0) && (ldb % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                                (reinterpret_cast<uintptr_t>(B) % 16 == 0);
            const bool tail_ok = big && vec_ok && opb == Op::N && !o.philox_b && o.epi == EPI_STORE &&
                                 !o.upper_tiles_only && tma_choice() && tail_choice();
            auto model = [&](int64_t s) {
                const int64_t kc = int64_t(ceil_div(ceil_div(K, int(s)), BK)) * BK;
                const double t_tile = 2.0 * BM * BN * double(kc) / cta_rate;
                if (s == 1 && tail_ok) {
                    const int64_t full = tiles / cap, ntail = tiles - full * cap;
                    const int64_t s_t = ntail > 0 ? std::min<int64_t>(8, cap / ntail) : 1;
                    if (full > 0 && ntail > 0 && s_t >= 2 && K >= 8 * kTBK * s_t)
                        return double(full) * t_tile + t_tile / double(s_t) +
                               2.0 * double(ntail * s_t) * BM * BN * 8.0 / hbm + 4e-6;
                }
                const int64_t waves = (tiles * s + cap - 1) / cap;
                double t = double(waves) * t_tile;
                if (s > 1) t += double(s + 1) * 8.0 * double(M) * N / hbm + 4e-6;
                return t;
            };
            // at most 64 splits, 512 MB of partials and k-chunks of >= 8 BK
            const int64_t ws_cap = (int64_t(512) << 20) / (8 * int64_t(M) * N + 1);
            const int64_t kmaxs = std::min<int64_t>(std::min<int64_t>(64, std::max<int64_t>(1, ws_cap)),
                                                    std::max<int64_t>(1, K / (8 * BK)));
            double best = model(1);
            for (int64_t s = 2; s <= kmaxs; ++s) {
                const double t = model(s);
                if (t < best * 0.995) {
                    best = t;
                    splits = int(s);
                }
            }
        }
    }
    int k_chunk = ceil_div(ceil_div(K, splits), BK) * BK;
    splits = ceil_div(K, k_chunk);
    p.k_chunk = k_chunk;
    p.splits = splits;

    const bool vec = (lda % 2 == 0) && (o.philox_b || ldb % 2 == 0) &&
                     (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                     (o.philox_b || reinterpret_cast<uintptr_t>(B) % 16 == 0);

    Buf ws, parts;
    int epi = o.epi;
    if (epi == EPI_STORE && splits > 1) {
        ws = Buf(ctx, sizeof(double) * size_t(splits) * M * N);
        p.ws = ws.d();
        epi = EPI_SPLIT;
    }
    if (epi == EPI_RESID) {
        parts = Buf(ctx, sizeof(double) * size_t(p.mt) * p.nt);
        p.partials = parts.d();
    }
    ProfScope prof(ctx, ctx.gemm_tag, M, N, K, 2.0 * M * double(N) * K);
    // TMA path: big tiles, B k-contiguous (op(B) = N) or generated, 16-byte
    // aligned operands with 16-byte-multiple leading dimensions
    const bool tma = big && vec && (opb == Op::N || o.philox_b) && tma_choice() && tensor_map_encoder();
    Buf tail_ws;
    int ntail = 0;
    if (tma && epi == EPI_STORE && splits == 1 && !o.philox_b && !o.upper_tiles_only && !o.tri_b_upper &&
        tail_choice()) {
        // the last partial wave runs its tiles as tail_split k-chunks each
        const int64_t full = (tiles / cap) * cap;
        ntail = int(tiles - full);
        const int s_t = ntail > 0 ? int(std::min<int64_t>(8, cap / ntail)) : 1;
        if (full > 0 && ntail > 0 && s_t >= 2 && K >= 8 * kTBK * s_t) {
            p.tail_base = int(full);
            p.tail_split = s_t;
            p.tail_kchunk = ceil_div(ceil_div(K, s_t), kTBK) * kTBK;
            tail_ws = Buf(ctx, sizeof(double) * size_t(ntail) * s_t * kTBM * kTBN);
            p.tail_ws = tail_ws.d();
        } else {
            ntail = 0;
        }
    }
    if (tma) {
        TmaPair maps;
        maps.a3d = 0;
        if (opa == Op::N && M % 16 == 0) {
            encode_map3_km(&maps.a, A, M, K, lda);            // A (M x K): one (16, BK, 8) box per stage
            maps.a3d = 1;
        } else if (opa == Op::N)
            encode_map(&maps.a, A, M, K, lda, 16, kTBK);      // A (M x K), eight 16-row boxes per stage
        else
            encode_map(&maps.a, A, K, M, lda, kTBK, kTBM);    // A^T: A is K x M, k-contiguous
        if (o.philox_b)
            maps.b = maps.a;
        else
            encode_map(&maps.b, B, K, N, ldb, kTBK, kTBN);    // B (K x N), k-contiguous
        if (opa == Op::N)
            launch_tma_epi<true>(ctx, p, maps, epi, o.philox_b);
        else
            launch_tma_epi<false>(ctx, p, maps, epi, o.philox_b);
        if (ntail > 0) {
            const int64_t tot = int64_t(ntail) * kTBM * kTBN;
            tail_reduce_kernel<<<int(std::min<int64_t>((tot + 255) / 256, int64_t(ctx.num_sms) * 8)), 256, 0,
                                 ctx.stream>>>(p.tail_ws, p.tail_split, p.tail_base, ntail, p.mt, p.nt, M, N, alpha,
                                               beta, C, ldc);
            RLRA_LAUNCH_CHECK();
            ++ctx.launches;
        }
    } else if (big && big_cfg_choice() == 16) {
        launch_ops<CfgBig16>(ctx, opa, opb, vec, p, epi, o.philox_b);
    } else if (big) {
        launch_ops<CfgBig>(ctx, opa, opb, vec, p, epi, o.philox_b);
    } else {
        launch_ops<CfgSmall>(ctx, opa, opb, vec, p, epi, o.philox_b);
    }

    if (epi == EPI_SPLIT) {
        const int64_t total = int64_t(M) * N;
        const int blocks = int(std::min<int64_t>((total + 255) / 256, int64_t(ctx.num_sms) * 8));
        split_reduce_kernel<<<blocks, 256, 0, ctx.stream>>>(p.ws, splits, M, N, alpha, beta, C, ldc,
                                                            o.upper_tiles_only ? 1 : 0, BM);
        RLRA_LAUNCH_CHECK();
        ++ctx.launches;
    }
    if (epi == EPI_RESID) sum_fixed_order(ctx, p.partials, int64_t(p.mt) * p.nt, o.resid_sq);
}

}  // namespace rlra_b200
