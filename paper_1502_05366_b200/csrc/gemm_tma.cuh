// gemm_tma.cuh — TMA-staged, warp-specialized FP64 DMMA GEMM (the big-tile
// path of gemm.cu: every product of the rsvd/QB/ID path whose operands are
// 16-byte aligned and whose B is k-contiguous, i.e. all products that stream
// A).
//
// One CTA computes a 128 x 128 tile of C = op(A) op(B):
//   * producer warpgroup: one elected thread issues cp.async.bulk.tensor (TMA)
//     loads of the A and B k-slices into a 6-stage shared-memory ring,
//     completing on the stage's "full" mbarrier (expect_tx bytes); for the
//     sketch the other producer threads generate the Philox Omega slice in
//     registers and store it into the same swizzled layout.  The sketch runs
//     as clusters of CL CTAs (CL m-tiles of one n-tile; CL = 2 by default):
//     each CTA generates 1/CL of the shared Omega slice and stores it into
//     every ring of the cluster with st.async (DSMEM), completing
//     transaction bytes on the peers' full mbarriers;
//   * 2 consumer warpgroups (8 warps of 64 x 32) read m8n8k4 fragments from
//     shared memory and issue DMMA.8x8x4; each warp releases the stage on its
//     "empty" mbarrier.
// Shared-memory tiles use the 128-byte TMA swizzle (16-byte chunk index XOR
// row index mod 8).  The fragment-row <-> matrix-row assignment is permuted so
// that every half-warp's 16 fragment loads hit 16 distinct bank pairs (the
// epilogue applies the same permutation when it writes C):
//   k-contiguous operand ("XM", rows of 16 k-values = 128 B): fragment rows
//     {0,2,4,6 | 1,3,5,7}, i.e. row(lr) = 2 (lr & 3) + (lr >> 2);
//   x-contiguous operand ("KM", A of Y = A Z: 8 boxes of 16 x-values x BK):
//     fragment f of a 16-row box takes rows
//     (lr & 1) + 8 ((lr >> 1) & 1) + 4 (lr >> 2) + 2 f.
#pragma once

#include <cuda.h>

#include "gemm.cuh"

namespace rlra_b200 {

struct TmaPair {
    CUtensorMap a;  // op(A) slices
    CUtensorMap b;  // B slices (unused for the Philox sketch)
    int a3d;        // A (x-contiguous) as a 3-D (16, K, M/16) map: one box per stage
};

constexpr int kTBM = 128, kTBN = 128, kTBK = 16, kTWM = 64, kTWN = 32, kTStages = 6;
constexpr int kTABytes = kTBM * kTBK * 8;  // 16 KB per stage
constexpr int kTBBytes = kTBN * kTBK * 8;  // 16 KB per stage
constexpr size_t kTmaSmem = size_t(kTStages) * (kTABytes + kTBBytes) + 1024;  // + 1 KB alignment slack

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
        "[%2];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// ---- cluster (DSMEM) helpers for the Omega-sharing sketch ----
__device__ __forceinline__ uint32_t cluster_map(uint32_t local_addr, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local_addr), "r"(rank));
    return r;
}
// asynchronous store into a cluster peer's shared memory that completes 16
// bytes of the peer's mbarrier transaction count (no fence needed: the data
// is visible once the barrier phase completes, as with TMA)
__device__ __forceinline__ void st_async_f64x2(uint32_t addr, double a, double b, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(addr),
                 "d"(a), "d"(b), "r"(remote_bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t remote_bar) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(remote_bar) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ double lds_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void lds_f64x2(uint32_t addr, double& a, double& b) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(a), "=d"(b) : "r"(addr));
}

// byte offset of element (k, x) in a swizzled stage tile
__device__ __forceinline__ uint32_t tma_km_off(int k, int x) {  // 8 boxes [BK][16 x]
    return uint32_t((x >> 4) * (kTBK * 128) + k * 128 + ((((x & 15) >> 1) ^ (k & 7)) << 4) + ((x & 1) << 3));
}
__device__ __forceinline__ uint32_t tma_xm_off(int k, int x) {  // [X][16 k] rows of 128 B
    return uint32_t(x * 128 + ((((k >> 1) ^ (x & 7))) << 4) + ((k & 1) << 3));
}
// fragment-row permutations (see header)
__device__ __forceinline__ int tma_xm_row(int lr) { return 2 * (lr & 3) + (lr >> 2); }
__device__ __forceinline__ int tma_km_row(int lr, int f) {
    return (lr & 1) + 8 * ((lr >> 1) & 1) + 4 * (lr >> 2) + 2 * f;
}
// Paired fragments (RLRA_GEMM_PAIRED, the default): every fragment load is a
// 16-byte ld.shared.v2.f64 that feeds two DMMAs.
//  * k-contiguous operands (B; A of A^T Y): the four k-steps of a 16-k stage
//    use k = 2 lc + 8 q + h (q, h in {0, 1}) instead of lc + 4 s, so a lane's
//    (k, k+1) sit in one 16-byte chunk; the rows of an 8-row fragment are
//    xm_row(lr) = (lr >> 1) + 4 (lr & 1), which puts the two lr of each 8-lane
//    phase in opposite chunk halves (conflict-free 16-byte loads);
//  * x-contiguous A (A Z): fragments 2p and 2p+1 of a 16-row box take rows
//    2 lr and 2 lr + 1, one 16-byte chunk; the chunk index is lr ^ (k & 7)
//    with k = 2 lc + 8 q + h, so the two lr of a phase (one even, one odd)
//    never share a chunk.
// The k-permutation is applied to both operands, so every k is summed once.
#ifndef RLRA_GEMM_PAIRED
#define RLRA_GEMM_PAIRED 1
#endif
__device__ __forceinline__ int tma_pi(int lr) { return (lr >> 1) + 4 * (lr & 1); }
__device__ __forceinline__ int xm_row(int lr) { return RLRA_GEMM_PAIRED ? tma_pi(lr) : tma_xm_row(lr); }
__device__ __forceinline__ int km_row(int lr, int f) { return RLRA_GEMM_PAIRED ? 2 * lr + f : tma_km_row(lr, f); }

template <bool A_KM, int EPI, bool PHILOX, int CL>
__global__ void __launch_bounds__(384, 1)
    dgemm_tma_kernel(const __grid_constant__ GemmParams p, const __grid_constant__ TmaPair maps) {
    static_assert(CL == 1 || PHILOX, "clusters share the generated Omega slice only");
    constexpr int NWM = kTBM / kTWM;  // 2
    constexpr int NCW = 8;            // consumer warps
    constexpr int MF = kTWM / 8, NF = kTWN / 8;
    extern __shared__ uint8_t tma_smem_raw[];
    // 1024-byte aligned ring (the 128-byte swizzle pattern repeats every 1 KB);
    // offsetting the __shared__ array keeps the shared address space, so the
    // fragment loads below compile to LDS, not generic loads
    uint8_t* smem = tma_smem_raw + ((1024u - (smem_u32(tma_smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + kTStages * kTABytes;
    __shared__ __align__(8) uint64_t full_bar[kTStages], empty_bar[kTStages];
    __shared__ double red[NCW];

    int tile = blockIdx.x;
    int nt_i, mt_i, split, crank = 0;
    int tpart = -1;  // >= 0: this CTA computes k-chunk tpart of a tail tile
    if (EPI == EPI_STORE && CL == 1 && tile >= p.tail_base) {
        const int q = tile - p.tail_base;
        tile = p.tail_base + q / p.tail_split;
        tpart = q % p.tail_split;
    }
    if (CL == 1) {
        nt_i = tile % p.nt;
        const int rest = tile / p.nt;
        mt_i = rest % p.mt;
        split = rest / p.mt;
        if (p.upper_tiles_only && mt_i > nt_i) return;
    } else {
        // clusters of CL consecutive m-tiles of one n-tile (the CTAs sharing
        // an Omega slice); the nt clusters of an m-group are adjacent so the
        // A rows they all read stay L2-resident.  m-tiles past mt are padding
        // CTAs: they generate their share of Omega, load zeros, store nothing.
        asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(crank));
        const int mg = (p.mt + CL - 1) / CL;
        const int q = tile / CL;
        nt_i = q % p.nt;
        const int rest = q / p.nt;
        mt_i = (rest % mg) * CL + (tile % CL);
        split = rest / mg;
    }
    const int m0 = mt_i * kTBM, n0 = nt_i * kTBN;
    int k_begin = split * p.k_chunk;
    int k_end = min(p.K, k_begin + p.k_chunk);
    if (tpart >= 0) {
        k_begin = tpart * p.tail_kchunk;
        k_end = min(p.K, k_begin + p.tail_kchunk);
    }
    if (p.tri_b_upper) k_end = min(k_end, n0 + kTBN);
    const int nk = k_end > k_begin ? (k_end - k_begin + kTBK - 1) / kTBK : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTStages; ++s) {
            // full: own expect_tx (+ the 4 Omega warps without a cluster; with
            // one, the peers' Omega stores complete transaction bytes);
            // empty: 8 consumer warps of every cluster CTA (a producer writes
            // the Omega slice into all of them)
            mbar_init(&full_bar[s], (PHILOX && CL == 1) ? 5u : 1u);
            mbar_init(&empty_bar[s], unsigned(NCW * CL));
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&maps.a)) : "memory");
        if (!PHILOX) asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&maps.b)) : "memory");
    }
    if (CL > 1)
        cluster_sync_all();  // every CTA's barriers exist before any remote arrive
    else
        __syncthreads();

    if (threadIdx.x < 128) {
        // ------------------------------------------------------ producer ---
        if (PHILOX)
            asm volatile("setmaxnreg.dec.sync.aligned.u32 96;\n");
        else
            asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n");
        if (!PHILOX && threadIdx.x != 0) return;
        uint32_t rb[CL], rbar[CL];  // the cluster CTAs' Omega rings and full barriers
#pragma unroll
        for (int r = 0; r < CL; ++r) {
            rb[r] = CL > 1 ? cluster_map(smem_u32(sB), r) : 0u;
            rbar[r] = CL > 1 ? cluster_map(smem_u32(&full_bar[0]), r) : 0u;
        }
        for (int kt = 0; kt < nk; ++kt) {
            const int st = kt % kTStages;
            if (kt >= kTStages) {
                mbar_wait(&empty_bar[st], ((kt / kTStages) - 1) & 1);
            }
            const int k0 = k_begin + kt * kTBK;
            uint8_t* a_st = sA + st * kTABytes;
            uint8_t* b_st = sB + st * kTBBytes;
            if (threadIdx.x == 0) {
                mbar_arrive_expect_tx(&full_bar[st], (PHILOX && CL == 1) ? unsigned(kTABytes)
                                                                          : unsigned(kTABytes + kTBBytes));
                if (A_KM) {
                    if (maps.a3d) {
                        // box (16, BK, 8) of the (16, K, M/16) view lands as
                        // [8][BK][16], the layout of the eight 2-D boxes
                        tma_load_3d(a_st, &maps.a, &full_bar[st], 0, k0, m0 / 16);
                    } else {
#pragma unroll
                        for (int b = 0; b < kTBM / 16; ++b)
                            tma_load_2d(a_st + b * (kTBK * 128), &maps.a, &full_bar[st], m0 + 16 * b, k0);
                    }
                } else {
                    tma_load_2d(a_st, &maps.a, &full_bar[st], k0, m0);
                }
                if (!PHILOX) tma_load_2d(b_st, &maps.b, &full_bar[st], k0, n0);
            }
            if (PHILOX) {
                // Omega(k, n) for this stage, 4 consecutive k of one column per
                // call; with a cluster each CTA generates 1/CL of the slice and
                // stores it into every cluster CTA's ring (DSMEM)
#pragma unroll
                for (int it = 0; it < (kTBN * kTBK / 4) / (128 * CL); ++it) {
                    const int g = (it * CL + crank) * 128 + threadIdx.x;
                    const int nl = g / (kTBK / 4), kl = (g % (kTBK / 4)) * 4;
                    const int n = n0 + nl, k = k0 + kl;
                    double v[4] = {0.0, 0.0, 0.0, 0.0};
                    if (n < p.N && k < k_end) {
                        philox_normal4(p.seed, p.draw, p.krow0 + k, n, v);
#pragma unroll
                        for (int t = 0; t < 4; ++t)
                            if (k + t >= k_end) v[t] = 0.0;
                    }
                    const uint32_t o0 = uint32_t(st * kTBBytes + nl * 128 + (((kl >> 1) ^ (nl & 7)) << 4));
                    const uint32_t o1 = uint32_t(st * kTBBytes + nl * 128 + ((((kl >> 1) + 1) ^ (nl & 7)) << 4));
                    if (CL == 1) {
                        uint8_t* row = b_st + nl * 128;
                        *reinterpret_cast<double2*>(row + ((((kl >> 1)) ^ (nl & 7)) << 4)) = make_double2(v[0], v[1]);
                        *reinterpret_cast<double2*>(row + ((((kl >> 1) + 1) ^ (nl & 7)) << 4)) =
                            make_double2(v[2], v[3]);
                    } else {
#pragma unroll
                        for (int r = 0; r < CL; ++r) {
                            st_async_f64x2(rb[r] + o0, v[0], v[1], rbar[r] + 8u * st);
                            st_async_f64x2(rb[r] + o1, v[2], v[3], rbar[r] + 8u * st);
                        }
                    }
                }
                if (CL == 1) {
                    __syncwarp();
                    if ((threadIdx.x & 31) == 0) mbar_arrive(&full_bar[st]);
                }
            }
        }
        if (CL > 1) cluster_sync_all();  // no CTA leaves while peers may still signal it
        return;
    }
    // -------------------------------------------------------- consumers ---
    if (PHILOX)
        asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n");
    else
        asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n");
    const int warp = (threadIdx.x >> 5) - 4, lane = threadIdx.x & 31;
    const int wm = warp % NWM, wn = warp / NWM;
    const int lr = lane >> 2, lc = lane & 3;
    int arow[MF], bcol[NF];
#pragma unroll
    for (int i = 0; i < MF; ++i)
        arow[i] = A_KM ? wm * kTWM + (i >> 1) * 16 + km_row(lr, i & 1) : wm * kTWM + i * 8 + xm_row(lr);
#pragma unroll
    for (int j = 0; j < NF; ++j) bcol[j] = wn * kTWN + j * 8 + xm_row(lr);
    // fragment byte offsets at kk = 0; the later k-steps are an XOR of the
    // swizzle bits (4..6) with a constant (+ a row immediate for KM):
    //   XM: off(kk) = off(0) ^ (kk << 3)
    //   KM: off(kk) = (off(0) ^ ((kk & 4) << 4)) + kk * 128
    //   paired: XM: off(q) = off(k0 = 2 lc) ^ (q << 6) (the (k, k+1) pair);
    //           KM: off(q, h) = (off(k0 = 2 lc) ^ (h << 4)) + (8 q + h) * 128
    constexpr int k0mul = RLRA_GEMM_PAIRED ? 2 : 1;
    uint32_t offa[MF], offb[NF];
#pragma unroll
    for (int i = 0; i < MF; ++i)
        offa[i] = A_KM ? tma_km_off(k0mul * lc, arow[i]) : tma_xm_off(k0mul * lc, arow[i]);
#pragma unroll
    for (int j = 0; j < NF; ++j) offb[j] = tma_xm_off(k0mul * lc, bcol[j]);

    double acc[MF][NF][2];
#pragma unroll
    for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    uint32_t rempty[CL];
#pragma unroll
    for (int r = 0; r < CL; ++r) rempty[r] = CL > 1 ? cluster_map(smem_u32(&empty_bar[0]), r) : 0u;
    const uint32_t sa0 = smem_u32(sA), sb0 = smem_u32(sB);
    int st = 0;
    uint32_t phase = 0;
    for (int kt = 0; kt < nk; ++kt) {
        mbar_wait(&full_bar[st], phase);
        const uint32_t a_s = sa0 + uint32_t(st * kTABytes);
        const uint32_t b_s = sb0 + uint32_t(st * kTBBytes);
        uint32_t fa[MF], fb[NF];
#pragma unroll
        for (int i = 0; i < MF; ++i) fa[i] = a_s + offa[i];
#pragma unroll
        for (int j = 0; j < NF; ++j) fb[j] = b_s + offb[j];
#if RLRA_GEMM_PAIRED
#pragma unroll
        for (int q = 0; q < kTBK / 8; ++q) {
            double af[2][MF], bf[2][NF];
            if (A_KM) {
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int i = 0; i < MF; i += 2)  // fa[i]: the even row, the chunk's first half
                        lds_f64x2((fa[i] ^ uint32_t(h << 4)) + uint32_t((8 * q + h) * 128), af[h][i], af[h][i + 1]);
            } else {
#pragma unroll
                for (int i = 0; i < MF; ++i) lds_f64x2(fa[i] ^ uint32_t(q << 6), af[0][i], af[1][i]);
            }
#pragma unroll
            for (int j = 0; j < NF; ++j) lds_f64x2(fb[j] ^ uint32_t(q << 6), bf[0][j], bf[1][j]);
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int i = 0; i < MF; ++i)
#pragma unroll
                    for (int j = 0; j < NF; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[h][i], bf[h][j]);
        }
#else
#pragma unroll
        for (int kk = 0; kk < kTBK; kk += 4) {
            double af[MF], bf[NF];
#pragma unroll
            for (int i = 0; i < MF; ++i)
                af[i] = A_KM ? lds_f64((fa[i] ^ uint32_t((kk & 4) << 4)) + uint32_t(kk * 128))
                             : lds_f64(fa[i] ^ uint32_t(kk << 3));
#pragma unroll
            for (int j = 0; j < NF; ++j) bf[j] = lds_f64(fb[j] ^ uint32_t(kk << 3));
#pragma unroll
            for (int i = 0; i < MF; ++i)
#pragma unroll
                for (int j = 0; j < NF; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
#endif
        __syncwarp();
        if (lane == 0) {
            if (CL == 1) {
                mbar_arrive(&empty_bar[st]);
            } else {
#pragma unroll
                for (int r = 0; r < CL; ++r) mbar_arrive_cluster(rempty[r] + 8u * st);
            }
        }
        if (++st == kTStages) {
            st = 0;
            phase ^= 1u;
        }
    }

    // ---------------------------------------------------------- epilogue ---
    // C element of acc[i][j][h]: row = arow[i] (this lane's lr), column = the
    // B-fragment row that lane (lr' = 2 lc + h) holds
    // EPI_RESID loads a group of two row fragments' R values first: C may
    // alias R (the in-place W <- W - Q_i B_i of the blocked QB), so loads left
    // inside the store loop would each wait a full memory round trip.  (The
    // other epilogues keep the plain loop: a load group there costs the
    // streaming kernels registers at the 168-register cap.)
    double local = 0.0;
    constexpr int RG = 2;  // row fragments per load group
#pragma unroll
    for (int i0 = 0; i0 < MF; i0 += RG) {
        double rin[RG][NF][2];
        if (EPI == EPI_RESID) {
#pragma unroll
            for (int ii = 0; ii < RG; ++ii) {
                const int row = m0 + arow[i0 + ii];
#pragma unroll
                for (int j = 0; j < NF; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int col = n0 + wn * kTWN + j * 8 + xm_row(2 * lc + h);
                        rin[ii][j][h] = (row < p.M && col < p.N) ? p.R[row + int64_t(col) * p.ldr] : 0.0;
                    }
            }
        }
#pragma unroll
        for (int ii = 0; ii < RG; ++ii) {
            const int i = i0 + ii;
            const int row = m0 + arow[i];
#pragma unroll
            for (int j = 0; j < NF; ++j) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int col = n0 + wn * kTWN + j * 8 + xm_row(2 * lc + h);
                    if (row < p.M && col < p.N) {
                        const double v = acc[i][j][h];
                        if (EPI == EPI_STORE && tpart >= 0) {
                            const int64_t slot = int64_t(tile - p.tail_base) * p.tail_split + tpart;
                            p.tail_ws[slot * (kTBM * kTBN) + (row - m0) + (col - n0) * kTBM] = v;
                        } else if (EPI == EPI_STORE) {
                            double* c = p.C + row + int64_t(col) * p.ldc;
                            *c = p.beta == 0.0 ? p.alpha * v : p.alpha * v + p.beta * *c;
                        } else if (EPI == EPI_SPLIT) {
                            p.ws[int64_t(split) * p.M * p.N + row + int64_t(col) * p.M] = v;
                        } else {
                            const double d = rin[ii][j][h] - p.alpha * v;
                            if (p.C) p.C[row + int64_t(col) * p.ldc] = d;
                            local += d * d;
                        }
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
    if (CL > 1) cluster_sync_all();
}

}  // namespace rlra_b200
