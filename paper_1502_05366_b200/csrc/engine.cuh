// engine.cuh — host orchestration of the randomized factorizations over the
// device kernels (reference L2: sketch.hpp, rsvd.hpp, qb.hpp, interp.hpp).
// All operands are device matrices; the C-ABI layer (capi.cu) handles host
// buffers, argument validation messages and status mapping.
#pragma once

#include <vector>

#include "common.cuh"

namespace rlra_b200 {

// Gaussian test-matrix source bound to one call (see rlra_omega in rlra_c.h).
struct OmegaSource {
    const rlra_omega* o = nullptr;
    int next_draw = 0;
};

// sketch.hpp:44-60 — Y (m x l)
// span_only: intermediate re-orthonormalisations keep the span but not an
// orthonormal basis (callers that never expose the sample).
// zpre (optional, with sketched): A^T Y of the sketch, accumulated while A
// was uploaded; the first power step then forms Z = (A^T Y) R^{-1} from the
// CholQR factor of Y instead of streaming A again (span-equal to A^T Q).
void sample_right(Context& ctx, const DMat& A, int l, int q, int s, OmegaSource& om, const DMat& Y,
                  bool span_only = false, bool sketched = false, const DMat* zpre = nullptr);

// Host-resident A: upload it into the device buffer dA in row chunks on the
// context's copy stream and compute the sketch Y = A Omega chunk by chunk as
// the rows land (the chunk GEMMs are the unchunked GEMM's tiles, so Y is
// bit-identical); consumes one Omega draw.
// With Zt (n x l) non-null and A large enough to upload in chunks, also
// Zt = A^T Y accumulated chunk by chunk (sum over the row chunks in order,
// under the upload): the first power product of rsvd (sample_right's zpre).
// Returns whether Zt was filled.
bool upload_and_sketch(Context& ctx, const double* hA, int64_t lda, const DMat& dA, int l, OmegaSource& om,
                       const DMat& Y, const DMat* Zt = nullptr);
// sketch.hpp:65-67 — returns Y^T (n x l) of the reference's l x n sample,
// computed on A directly (the reference materialises A^T; we never do).
void sample_left_t(Context& ctx, const DMat& A, int l, int q, int s, OmegaSource& om, const DMat& Yt,
                   bool span_only = false);

// Y = A Omega (op(A) = A or A^T), one Omega draw from om
enum class Op;
void sketch(Context& ctx, Op op_a, const DMat& A, int l, OmegaSource& om, const DMat& Y);
// Y (M x l) = op(A) * Omega, Omega the K x l Philox draw starting at row
// krow0 of the stream (materialised, or in-GEMM with RLRA_SKETCH_FUSED=1)
void sketch_philox(Context& ctx, Op op_a, int M, int l, int K, const double* A, int64_t lda, uint64_t seed, int draw,
                   int64_t krow0, double* Y, int64_t ldy);

// rsvd.hpp:144-156 finish_qb_qr_bt: Q m x l, Bt n x l (overwritten by Qhat)
void finish_qr_bt(Context& ctx, const DMat& Q, const DMat& Bt, int k, const DMat& U, double* sigma,
                  const DMat& V);

// rsvd.hpp:127-160; U m x k, sigma (device) k, V n x k
void rsvd(Context& ctx, int variant, const DMat& A, int k, int p, int q, int s, OmegaSource& om,
          const DMat& U, double* sigma, const DMat& V, const DMat* sketched = nullptr,
          const DMat* zpre = nullptr);

struct QbOut {
    int ell = 0;
    std::vector<double> hist;
    double final_residual = 0.0;
    bool reached = true;
};
// qb.hpp:98-142 on W (destroyed: left as A - QB).  Q m x cap, B cap x n.
QbOut qb_blocked(Context& ctx, const DMat& W, int blk, int num_blocks, double tol, int q_power,
                 int reorth_period, OmegaSource& om, const DMat& Q, const DMat& B);

// qb.hpp:159-204 / 211-271 (the composite drivers); Q m x (b*M), B (b*M) x n;
// Omega draw ids (node << 16) | block.  Return ||A - QB||_F.
double qb_parallel(Context& ctx, const DMat& A, int blk, int num_blocks, int q_power, OmegaSource& om, const DMat& Q,
                   const DMat& B);
double qb_hierarchical(Context& ctx, const DMat& A, int num_row_blocks, int blk, int num_blocks, int q_power,
                       OmegaSource& om, const DMat& Q, const DMat& B);

// qb.hpp:276-288 (k already resolved to [1, ell]); U m x k, sigma k, V n x k
void svd_from_qb(Context& ctx, const DMat& Q, const DMat& B, int k, int vnum, const DMat& U,
                 double* sigma, const DMat& V);

struct IdOut {
    int k = 0;
    double qr_residual = 0.0;
    bool reached = true;
    bool clamped = false;
};
// interp.hpp:101-104 — jc (device, n), V (n x kmax)
IdOut id_column(Context& ctx, const DMat& A, int k, double tol, int* jc, const DMat& V);
// interp.hpp:203-223 — jc (device, n), V (n x k)
IdOut id_rand(Context& ctx, const DMat& A, int k, int p, int q, int s, OmegaSource& om, int* jc,
              const DMat& V);
// interp.hpp:123-140 — jr (device, m), Wr (m x k)
void two_sided_from_column(Context& ctx, const DMat& A, const int* jc, int k, int* jr, const DMat& Wr);
// interp.hpp:143-177 — C m x k, U k x k, R k x n; returns ||A - CUR||_F
double cur_from_two_sided(Context& ctx, const DMat& A, const int* jc, const int* jr, const DMat& V,
                          int k, const DMat& C, const DMat& U, const DMat& R, const int* jr_host);

// interp.hpp:143-156 — U (k x k) from the skeleton rows R (k x n) and V (n x k)
void cur_linkage(Context& ctx, const DMat& R, const DMat& V, int k, const DMat& U, const int* jr_host);

// ||A||_F (device-side deterministic reduction, read back)
double frobenius(Context& ctx, const DMat& A);

// scatter V = P [I_k; T^T] (interp.hpp:65-72)
void build_interp(Context& ctx, const int* perm, const DMat& T, int n, int k, const DMat& V);

}  // namespace rlra_b200
