/*
 * rlra_c.h — C-ABI of the B200 engine for the reference's randomized
 * low-rank factorization path (the drop-in boundary).
 *
 * The reference ("rlra", /root/reference/proj/include/rlra) is a header-only
 * C++20 library whose operator API is the free functions of namespace rlra.
 * It has no C ABI of its own; the functions below are what a binding of that
 * API needs, one entry point per reference function on the hot path
 * (SURVEY.md §8b).  include/rlra/<name>.hpp re-declares the reference API with the
 * exact signatures and implements it over this header, so C++ callers switch
 * by changing the include path; INTEGRATION.md shows the ctypes binding.
 *
 * Conventions (reference core/matrix.hpp:17-80):
 *   - matrices are column-major float64, element (i,j) at p[i + j*ld];
 *   - every matrix argument is (pointer, rows, cols, ld) and `loc` says whether
 *     the pointers are host (RLRA_HOST) or device (RLRA_DEVICE) memory; host
 *     inputs are copied to the device, outputs copied back, inside the call;
 *   - output buffers are caller-allocated; sizes are stated per function;
 *   - all arithmetic is FP64 on hand-written sm_100a kernels; nothing falls
 *     back to the CPU, cuBLAS or cuSOLVER.  A missing device is RLRA_ECUDA.
 *
 * Errors: every function returns rlra_status.  The statuses map 1:1 onto the
 * reference exception classes (core/errors.hpp:11-33) and the message, which
 * reproduces the reference's text where the reference's tests match on it,
 * is available from rlra_last_error() (thread-local, valid until the next
 * failing call on the same thread).
 *
 * Threading: a context is used by one host thread at a time.
 */
#ifndef RLRA_C_H
#define RLRA_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RLRA_OK = 0,
    RLRA_EDIM = 1,   /* rlra::DimensionError   core/errors.hpp:16-18 */
    RLRA_ENUM = 2,   /* rlra::NumericalError   core/errors.hpp:21-23 */
    RLRA_ECONV = 3,  /* rlra::ConvergenceError core/errors.hpp:26-28 */
    RLRA_EIO = 4,    /* rlra::IoError          core/errors.hpp:31-33 */
    RLRA_ECUDA = 5,  /* CUDA failure / no device -> rlra::Error */
    RLRA_ENCCL = 6,  /* collective failure       -> rlra::Error */
    RLRA_EINVAL = 7  /* bad handle or argument   -> rlra::Error */
} rlra_status;

enum { RLRA_HOST = 0, RLRA_DEVICE = 1 };

/* rsvd variants: rsvd.hpp:154 (v2, QR of B^T), :144 (v1, B B^T), :127 (basic) */
enum { RLRA_RSVD_V2 = 0, RLRA_RSVD_V1 = 1, RLRA_RSVD_BASIC = 2 };
/* Vnum (sketch.hpp:14) */
enum { RLRA_VNUM_QR = 0, RLRA_VNUM_BBT = 1 };

typedef struct rlra_ctx rlra_ctx;

/* ---------------------------------------------------------------- Omega ---
 * Where the Gaussian test matrices come from.
 *  RLRA_OMEGA_CALLBACK (parity mode): the engine calls fill(user, draw, rows,
 *    cols, host_out) once per Gaussian draw, in the reference's order, and
 *    uploads the result.  The C++ shim implements fill with the caller's
 *    rlra::RngState (core/rng.hpp), so the draws and the post-call RNG state
 *    are the reference's bit for bit.  Draw order:
 *      rsvd_*      : one n x l draw                    (sketch.hpp:51, rsvd.hpp:130)
 *      sample_left : one m x l draw                    (sketch.hpp:51,66)
 *      id_rand / cur_rand : one m x l draw             (interp.hpp:208)
 *      qb_blocked  : draw i = block i, n x width_i; the callback performs the
 *                    per-block rng.substream() itself  (qb.hpp:119-120)
 *  RLRA_OMEGA_PHILOX (performance mode): entries are Philox4x32-10 normals
 *    keyed by `seed` (counter = row, column, draw), identical on every GPU of
 *    a row-sharded run.  By default Omega is generated once per call into an
 *    n x l device buffer (82 MB at C5: 0.25% of A's bytes) that the streaming
 *    GEMM reads; RLRA_SKETCH_FUSED=1 generates it in-register inside the
 *    GEMM's producer warps instead (never in HBM, the same bits), which
 *    measured slower at C5 (122.8 vs 115.7 ms: every cluster of M-tiles
 *    regenerates its slice).  The caller's RNG is not
 *    consumed by the engine (the shim derives `seed` from one next_u64()). */
enum { RLRA_OMEGA_CALLBACK = 0, RLRA_OMEGA_PHILOX = 1 };
typedef void (*rlra_omega_fill_fn)(void* user, int draw, int rows, int cols, double* host_out);
typedef struct {
    int mode;
    rlra_omega_fill_fn fill;
    void* user;
    uint64_t seed;
} rlra_omega;

/* -------------------------------------------------- reference RNG stream ---
 * The reference's RngState (core/rng.hpp:18-79): xoshiro256++ seeded by
 * splitmix64, Box-Muller through libm with a cached spare, column-major
 * fills.  Host code, bit-identical to the reference on the same libm; it
 * exists so parity-mode callers without the C++ shim (ctypes, the CLI) can
 * produce the reference's Omega.  Field order matches the reference class. */
typedef struct {
    uint64_t s[4];
    double spare;
    int have_spare;
} rlra_rng;
void rlra_rng_seed(rlra_rng* r, uint64_t seed);
uint64_t rlra_rng_next_u64(rlra_rng* r);
double rlra_rng_next_gaussian(rlra_rng* r);
void rlra_rng_substream(rlra_rng* parent, rlra_rng* child);
void rlra_rng_gaussian_fill(rlra_rng* r, int rows, int cols, double* out);
/* rlra_omega.fill callbacks with user = rlra_rng*: a plain draw
 * (rsvd/sample/id_rand) and substream-then-draw (qb_blocked, qb.hpp:119). */
void rlra_omega_fill_rng(void* user, int draw, int rows, int cols, double* out);
void rlra_omega_fill_rng_substream(void* user, int draw, int rows, int cols, double* out);
/* Per-node streams for the composite QB drivers (qb_parallel, qb_hierarchical):
 * draw ids are (node << 16) | block; nodes[node] is the node's RngState in the
 * reference's order (qb_parallel: one substream per block, drawn directly;
 * qb_hierarchical: the leaf substreams then the merge substreams, each
 * node's qb_blocked taking one further substream per block). */
typedef struct {
    rlra_rng* nodes;
    int count;
    int substream_per_draw;
} rlra_rng_nodes;
void rlra_omega_fill_rng_nodes(void* user, int draw, int rows, int cols, double* out);

/* ------------------------------------------------------------- context --- */
rlra_status rlra_ctx_create(int device, rlra_ctx** out);
rlra_status rlra_ctx_destroy(rlra_ctx* ctx);
rlra_status rlra_ctx_synchronize(rlra_ctx* ctx);
/* Number of engine kernel launches issued on this context so far. */
uint64_t rlra_ctx_launch_count(const rlra_ctx* ctx);
/* Optional timing: when enabled every engine GEMM launch and every phase
 * (orth, small_svd, cpqr) is bracketed by CUDA events on the context stream.
 * Enabling or disabling clears the records. */
rlra_status rlra_ctx_profile(rlra_ctx* ctx, int enable);
int rlra_ctx_profile_count(const rlra_ctx* ctx);
rlra_status rlra_ctx_profile_get(rlra_ctx* ctx, int i, char* name, int name_cap, int* M, int* N,
                                 int* K, double* flops, double* ms);
/* The cudaStream_t the context launches on (for event timing by callers). */
void* rlra_ctx_stream(const rlra_ctx* ctx);
const char* rlra_last_error(void);

/* qb_parallel (qb.hpp:159-204): M independent block samples, per-block
 * orthonormalisation, sequential cross-block projection, B = Q^T A, ell = b*M.
 * qb_hierarchical (qb.hpp:211-271): fixed-rank QB of num_row_blocks (2^j)
 * horizontal slabs, merged pairwise up a binary tree (QB of the stacked B's,
 * Q lifted through the block-diagonal stages).  q: m x (b*M), b: (b*M) x n.
 * Omega draw ids: (node << 16) | block (see rlra_rng_nodes). */
rlra_status rlra_qb_parallel(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda, int blk,
                             int num_blocks, int q_power, const rlra_omega* omega, double* q, int64_t ldq,
                             double* b, int64_t ldb, double* final_residual);
rlra_status rlra_qb_hierarchical(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda,
                                 int num_row_blocks, int blk, int num_blocks, int q_power, const rlra_omega* omega,
                                 double* q, int64_t ldq, double* b, int64_t ldb, double* final_residual);

/* qb_single (qb.hpp:43-95): one direction at a time until ||A - QB||_F < tol
 * or max_rank columns; q m x max_rank, b max_rank x n (ld >= max_rank); Omega
 * draws are n x 1 columns in the reference's order (redraws included). */
rlra_status rlra_qb_single(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda, double tol,
                           int max_rank, const rlra_omega* omega, double* q, int64_t ldq, double* b, int64_t ldb,
                           int* ell, double* hist, int* nhist, double* final_residual, int* reached);

/* ------------------------------------------- I/O, generator, verifier ---
 * Binary matrix files in the reference format (io.hpp:40-109): int32 rows,
 * int32 cols (little-endian), then rows*cols doubles row by row; exactly
 * 8 + 8*rows*cols bytes; every value finite.  Errors are RLRA_EIO with the
 * reference's messages.  rlra_load_binary reads rows [row0, row0 + rows) — a
 * row shard — into a column-major (host or device) buffer, transposing on the
 * GPU as the chunks stream in. */
rlra_status rlra_binary_header(const char* path, int* rows, int* cols);
rlra_status rlra_load_binary(rlra_ctx* ctx, int loc, const char* path, int64_t row0, int rows, double* a, int64_t lda);
rlra_status rlra_save_binary(rlra_ctx* ctx, int loc, const char* path, const double* a, int m, int n, int64_t lda);
/* gen_test_matrix (testmat.hpp:65-74): A = U diag(sigma[0..r)) V^T + noise*G
 * with U, V orthonormalised Philox Gaussians of `seed` (not the reference's
 * RngState bits; the spectrum is what the configs specify). */
rlra_status rlra_gen_test_matrix(rlra_ctx* ctx, int loc, int m, int n, const double* sigma, int r, uint64_t seed,
                                 double noise, double* a, int64_t lda);
/* verify(a, SvdFactors, sigma_true) (report.hpp:97-138): out[0] relative
 * Frobenius error, out[1] relative spectral error (60-step power estimates,
 * start vectors from RngState 0x5bd1e995 as the reference), out[2..4] the
 * Frobenius floor, spectral floor and sketch bound (NaN without sigma_true,
 * r = 0). */
/* verify_reconstruction (report.hpp:97-138) for recon = X Y^T (X m x k,
 * Y n x k): the ID (X = C, Y = V), CUR (X = C, Y = (U R)^T) and QB (X = Q,
 * Y = B^T) reports.  out as rlra_verify_svd. */
rlra_status rlra_verify_lowrank(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda, const double* x,
                                int64_t ldx, const double* y, int64_t ldy, int k, const double* sigma_true, int r,
                                double out[5]);
rlra_status rlra_verify_svd(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda, const double* u,
                            int64_t ldu, const double* sigma, const double* v, int64_t ldv, int k,
                            const double* sigma_true, int r, double out[5]);

/* ------------------------------------------------- row-sharded multi-GPU ---
 * One process (one rlra_ctx) per GPU; A (m_total x n) split by rows.  The
 * collectives are NCCL (loaded at run time from libnccl.so.2) on the context
 * stream over NVLink: allreduce of the l x l CholQR Grams and of the n x l
 * partials A^T Y / A^T Q (BASELINE north_star).  Launcher: rank 0 calls
 * rlra_comm_unique_id and distributes the 128 bytes (MPI, torch.distributed,
 * a file); every rank calls rlra_comm_create with its rank.  Replaces the
 * reference's single-address-space rsvd_v2 (rsvd.hpp:154-160) for
 * multi-GPU callers; single-GPU callers keep rlra_rsvd. */
typedef struct rlra_comm rlra_comm;
rlra_status rlra_comm_unique_id(unsigned char id[128]);
rlra_status rlra_comm_create(rlra_ctx* ctx, const unsigned char id[128], int nranks, int rank, rlra_comm** out);
rlra_status rlra_comm_destroy(rlra_comm* comm);
/* Host-staged collectives: the same drivers over collectives the caller
 * supplies (MPI, gloo, shared memory, ...).  Each exchanged buffer is copied
 * to pinned host memory after the context stream drains, combined by these
 * functions (0 = success; anything else fails the call with RLRA_ENCCL), and
 * copied back, so no kernel of one rank ever waits on another rank.
 *   allreduce_sum: in-place elementwise sum of count doubles over the ranks;
 *                  every rank must receive the same bits.
 *   allgather:     recv[r * count + i] = rank r's send[i].
 *   gpu_acquire / gpu_release (both or neither): a token held while this
 *                  rank's GPU work is in flight; the drivers release it while
 *                  they wait in a collective.  Ranks sharing one GPU use it to
 *                  keep one rank's kernels on the device at a time. */
typedef struct rlra_host_collectives {
    int (*allreduce_sum)(void* user, double* buf, size_t count);
    int (*allgather)(void* user, const double* send, double* recv, size_t count);
    void (*gpu_acquire)(void* user);
    void (*gpu_release)(void* user);
    void* user;
} rlra_host_collectives;
rlra_status rlra_comm_create_host(rlra_ctx* ctx, int nranks, int rank, const rlra_host_collectives* coll,
                                  rlra_comm** out);
/* An in-process group of nranks ranks run as threads (one rlra_ctx each):
 * shared-memory collectives (sums formed in rank order on every rank), a
 * barrier that fails with RLRA_ENCCL after timeout_s (<= 0: the
 * RLRA_COMM_TIMEOUT_S default, 600 s) instead of hanging, and a GPU token. */
typedef struct rlra_local_group rlra_local_group;
rlra_status rlra_local_group_create(int nranks, double timeout_s, rlra_local_group** out);
rlra_status rlra_local_group_collectives(rlra_local_group* g, int rank, rlra_host_collectives* out);
rlra_status rlra_local_group_destroy(rlra_local_group* g);
/* Failure detection (NCCL communicators): waits poll ncclCommGetAsyncError and
 * abort the communicator (ncclCommAbort) on an asynchronous error or after
 * RLRA_COMM_TIMEOUT_S seconds (default 600), failing with RLRA_ENCCL instead of
 * hanging.  NCCL_ALGO=Ring and NCCL_PROTO=Simple are pinned (unless set) so the
 * reduction order, and every replicated factor, is fixed run to run. */
/* Rows [row0, row0 + m_local) of the rlra_gen_test_matrix matrix (testmat.hpp:
 * 65-74 semantics) of an m_total x n A: U's Philox rows are orthonormalised
 * across the ranks (distributed CholQR2), V replicated; equal to the
 * single-GPU generator's rows up to rounding. */
rlra_status rlra_gen_test_matrix_rowsharded(rlra_ctx* ctx, rlra_comm* comm, int loc, int64_t row0, int m_local,
                                            int64_t m_total, int n, const double* sigma, int r, uint64_t seed,
                                            double noise, double* a, int64_t lda);
/* rsvd_v2 with A's rows [row0, row0 + m_local) on this rank (a: m_local x n,
 * loc host or device); U: this rank's m_local x k rows of U; sigma (k) and V
 * (n x k) replicated.  Omega: Philox (identical on every rank) or a callback
 * that draws the same n x l matrix on every rank. */
/* id_rand (interp.hpp:203-223) with A row-sharded: jc (n, 0-based column
 * permutation, first k the skeleton) and V (n x k) replicated; the sketch is
 * an allreduce of n x l partials.  Omega~ is m_total x l (Philox counter =
 * global row), this rank using rows [row0, row0 + m_local). */
rlra_status rlra_id_rand_rowsharded(rlra_ctx* ctx, rlra_comm* comm, int loc, const double* a, int m_local, int n,
                                    int64_t lda, int64_t row0, int64_t m_total, int k, int p, int q, int s,
                                    const rlra_omega* omega, int* jc, double* v, int64_t ldv,
                                    double* qr_residual, int* clamped);
/* cur_rand (interp.hpp:240-244) with A row-sharded: the row ID of C = A(:,Jc)
 * is a column-pivoted QR whose pivot statistics are allgathered each step
 * (north_star).  jc, v (n x k), jr (k global rows), u (k x k), r (k x n)
 * replicated; w (m_local x k) and c (m_local x k) this rank's rows;
 * residual = ||A - C U R||_F over all ranks. */
rlra_status rlra_cur_rand_rowsharded(rlra_ctx* ctx, rlra_comm* comm, int loc, const double* a, int m_local, int n,
                                     int64_t lda, int64_t row0, int64_t m_total, int k, int p, int q, int s,
                                     const rlra_omega* omega, int* jc, int* jr, double* v, int64_t ldv, double* w,
                                     int64_t ldw, double* c, int64_t ldc, double* u, int64_t ldu, double* r,
                                     int64_t ldr, double* residual, double* qr_residual);
/* qb_blocked (qb.hpp:98-152) with W row-sharded (this rank's m_local rows;
 * destroyed when inplace on the device, else copied): q (m_local x cap) this
 * rank's rows of Q, b (cap x n) replicated; ell, residual history, final
 * residual and tolerance flag as rlra_qb_blocked.  rlra_svd_from_qb on
 * (q, b) with m = m_local then yields this rank's rows of U. */
rlra_status rlra_qb_blocked_rowsharded(rlra_ctx* ctx, rlra_comm* comm, int loc, double* a, int m_local, int n,
                                       int64_t lda, int64_t m_total, int inplace, int blk, int num_blocks,
                                       double tol, int q_power, int reorth_period, const rlra_omega* omega,
                                       double* q, int64_t ldq, double* b, int64_t ldb, int cap, int* ell,
                                       double* hist, int* nhist, double* final_residual, int* reached);
/* qb_hierarchical (qb.hpp:211-271) over the ranks: num_row_blocks = world * L
 * (a power of two), rank g holding slabs [g L, (g+1) L) of the reference's
 * partition (floor(m_total / num_row_blocks) rows each, the last slab the
 * remainder).  Leaves and the rank's own subtree merge locally; the subtree
 * roots' B are allgathered over NVLink and the upper merges run replicated.
 * q: this rank's m_local x (b*M) rows of Q, b: (b*M) x n replicated. */
rlra_status rlra_qb_hierarchical_rowsharded(rlra_ctx* ctx, rlra_comm* comm, int loc, const double* a, int m_local,
                                            int n, int64_t lda, int64_t m_total, int num_row_blocks, int blk,
                                            int num_blocks, int q_power, const rlra_omega* omega, double* q,
                                            int64_t ldq, double* b, int64_t ldb, double* final_residual);
/* rsvd_v2 (rsvd.hpp:154-160) with A row-sharded over the ranks: rank g holds
 * m_local rows of the m_total x n matrix; the Grams and the n x l partials
 * A_g^T Y_g are allreduced (the north_star exchange), the l x l work is
 * replicated.  u: this rank's m_local x k rows of U; sigma, v replicated.
 * loc = RLRA_HOST: the shard is uploaded in row chunks under the local
 * sketch GEMM (as rlra_rsvd does for a host A). */
rlra_status rlra_rsvd_rowsharded(rlra_ctx* ctx, rlra_comm* comm, int loc, const double* a, int m_local, int n,
                                 int64_t lda, int64_t m_total, int k, int p, int q, int s,
                                 const rlra_omega* omega, double* u, int64_t ldu, double* sigma, double* v,
                                 int64_t ldv);
const char* rlra_version(void);

/* -------------------------------------------------------- kernel level --- */
/* core/matmul.hpp:68: c (m x n) = op(a) * op(b); a is ar x ac, b is br x bc. */
rlra_status rlra_matmul(rlra_ctx* ctx, int loc, int trans_a, int trans_b, const double* a, int ar,
                        int ac, int64_t lda, const double* b, int br, int bc, int64_t ldb,
                        double* c, int64_t ldc);

/* core/qr.hpp:95: a (m x n, m >= n) = q (m x n) * r (n x n), diag(r) >= 0.
 * r may be NULL (orth, core/qr.hpp:125).  degenerate may be NULL. */
rlra_status rlra_compact_qr(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda,
                            double* q, int64_t ldq, double* r, int64_t ldr, int* degenerate);

/* core/qr.hpp:140: partial column-pivoted QR.  kmax = k (rank mode) or
 * min(m,n) (k == 0, tol > 0).  q1 (m x kmax, may be NULL), s1 (kmax x n),
 * perm (n ints).  Rows/columns past *frank are left untouched. */
rlra_status rlra_pivoted_qr(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda,
                            int k, double tol, double* q1, int64_t ldq1, double* s1,
                            int64_t lds1, int* perm, int* frank, double* residual, int* reached,
                            int* degenerate);

/* core/qr.hpp:242: t (k x nc) = s11^{-1} s12 with the 1e12 / 1e4 clamp. */
rlra_status rlra_upper_tri_solve(rlra_ctx* ctx, int loc, const double* s11, int k, int64_t lds11,
                                 const double* s12, int nc, int64_t lds12, double* t,
                                 int64_t ldt, int* clamped);

/* core/jacobi.hpp:145: r = min(m,n); u (m x r), sigma (r), v (n x r). */
rlra_status rlra_small_svd(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda,
                           double* u, int64_t ldu, double* sigma, double* v, int64_t ldv);

/* core/jacobi.hpp:68: values (n, descending), vectors (n x n). */
rlra_status rlra_sym_eig(rlra_ctx* ctx, int loc, const double* t, int n, int64_t ldt,
                         double* values, double* vectors, int64_t ldv);

/* core/norms.hpp:29 */
rlra_status rlra_frobenius_norm(rlra_ctx* ctx, int loc, const double* a, int m, int n,
                                int64_t lda, double* out);

/* ------------------------------------------ row-sharded building blocks ---
 * The multi-GPU path (paper_1502_05366_b200/dist.py) row-shards A across
 * ranks and runs these per-shard steps between NCCL collectives: the sketch
 * with a global row offset (so every rank sees the same Philox Omega), the
 * local Gram of a CholQR pass, the replicated Cholesky + inverse of the
 * allreduced Gram, and the local triangular update. */

/* Y = op(A) * Omega_draw.  trans = 0: A m x n, Omega n x l, Y m x l;
 * trans = 1: A m x n, Omega m x l (rows row0.. of the global Omega), Y n x l. */
rlra_status rlra_sketch(rlra_ctx* ctx, int loc, int trans, const double* a, int m, int n,
                        int64_t lda, int l, const rlra_omega* omega, int draw, int64_t row0,
                        double* y, int64_t ldy);

/* G = Y^T Y (n x n, full symmetric) for Y m x n. */
rlra_status rlra_gram(rlra_ctx* ctx, int loc, const double* y, int m, int n, int64_t ldy,
                      double* g, int64_t ldg);

/* Upper Cholesky G = R^T R and R^{-1} (both n x n, strictly lower parts 0).
 * *ok = 0 when a pivot falls below floor * (original diagonal); then R and
 * Rinv are unusable.  G is not modified. */
rlra_status rlra_chol_inv(rlra_ctx* ctx, int loc, const double* g, int n, int64_t ldg,
                          double floor, double* r, int64_t ldr, double* rinv, int64_t ldri,
                          int* ok);

/* out = Y * T for Y (m x n) and upper-triangular T (n x n); out may not
 * alias Y. */
rlra_status rlra_trmm_right_upper(rlra_ctx* ctx, int loc, const double* y, int m, int n,
                                  int64_t ldy, const double* t, int64_t ldt, double* out,
                                  int64_t ldo);

/* ||A - X Y^T||_F for A (m x n), X (m x k), Y (n x k): the dense
 * reconstruction residual of report.hpp:97-113 (and of the CUR residual,
 * interp.hpp:175) as one fused GEMM + subtract + sum-of-squares pass that
 * never materialises X Y^T. */
rlra_status rlra_lowrank_residual(rlra_ctx* ctx, int loc, const double* a, int m, int n,
                                  int64_t lda, const double* x, int64_t ldx, const double* y,
                                  int64_t ldy, int k, double* out);

/* Materialise the Philox Omega the sketch GEMM generates in-register
 * (rows x cols, draw index `draw`, row offset `row0`).  Test/diagnostic use. */
rlra_status rlra_gaussian_philox(rlra_ctx* ctx, int loc, int rows, int cols, uint64_t seed,
                                 int draw, int64_t row0, double* out, int64_t ld);

/* ---------------------------------------------------------- algorithms --- */
/* sketch.hpp:44 (left=0, y m x l) and sketch.hpp:65 (left=1, y l x n). */
rlra_status rlra_sample(rlra_ctx* ctx, int loc, int left, const double* a, int m, int n,
                        int64_t lda, int l, int q, int s, const rlra_omega* omega, double* y,
                        int64_t ldy);

/* rsvd.hpp:127/144/154.  u (m x k), sigma (k), v (n x k). */
rlra_status rlra_rsvd(rlra_ctx* ctx, int loc, int variant, const double* a, int m, int n,
                      int64_t lda, int k, int p, int q, int s, const rlra_omega* omega, double* u,
                      int64_t ldu, double* sigma, double* v, int64_t ldv);

/* qb.hpp:98/148.  If inplace, `a` is overwritten with A - QB
 * (qb_blocked_inplace); otherwise it is read only.  q (m x cap), b (cap x n)
 * with cap >= min(blk*num_blocks, min(m,n)); hist has num_blocks entries. */
rlra_status rlra_qb_blocked(rlra_ctx* ctx, int loc, double* a, int m, int n, int64_t lda,
                            int inplace, int blk, int num_blocks, double tol, int q_power,
                            int reorth_period, const rlra_omega* omega, double* q, int64_t ldq,
                            double* b, int64_t ldb, int cap, int* ell, double* hist, int* nhist,
                            double* final_residual, int* reached);

/* qb.hpp:276.  q (m x ell), b (ell x n).  k == 0 keeps all ell.
 * u (m x k_out), sigma (k_out), v (n x k_out); size them for k or ell. */
rlra_status rlra_svd_from_qb(rlra_ctx* ctx, int loc, const double* q, int m, int64_t ldq,
                             const double* b, int n, int64_t ldb, int ell, int k, int vnum,
                             double* u, int64_t ldu, double* sigma, double* v, int64_t ldv,
                             int* k_out);

/* interp.hpp:101: column ID, rank (k >= 1, tol == 0) or tolerance mode
 * (k == 0, tol > 0).  jc (n), v (n x kmax). */
rlra_status rlra_id_column(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda,
                           int k, double tol, int* jc, double* v, int64_t ldv, int* k_out,
                           double* qr_residual, int* reached, int* clamped);

/* interp.hpp:203: jc (n), v (n x k). */
rlra_status rlra_id_rand(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda,
                         int k, int p, int q, int s, const rlra_omega* omega, int* jc, double* v,
                         int64_t ldv, double* qr_residual, int* clamped);

/* interp.hpp:123: row side of a finished column ID of rank k.  jr (m),
 * w (m x k). */
rlra_status rlra_two_sided_from_column(rlra_ctx* ctx, int loc, const double* a, int m, int n,
                                       int64_t lda, const int* jc, int k, int* jr, double* w,
                                       int64_t ldw);

/* interp.hpp:158: c (m x k), u (k x k), r (k x n), residual = ||A - CUR||_F. */
rlra_status rlra_cur_from_two_sided(rlra_ctx* ctx, int loc, const double* a, int m, int n,
                                    int64_t lda, const int* jc, const int* jr, const double* v,
                                    int64_t ldv, int k, double* c, int64_t ldc, double* u,
                                    int64_t ldu, double* r, int64_t ldr, double* residual);

/* interp.hpp:143-156 (rlra::detail::cur_linkage): u (k x k) =
 * argmin ||U R - V^T||_F via a compact QR of R^T, for r (k x n) and v (n x k).
 * jr: at least k HOST ints (the skeleton rows, named in the NumericalError
 * when R is rank-deficient to working precision: |R^(i,i)| < 1e-13 max). */
rlra_status rlra_cur_linkage(rlra_ctx* ctx, int loc, const double* r, int k, int n, int64_t ldr,
                             const double* v, int64_t ldv, const int* jr, double* u, int64_t ldu);

/* interp.hpp:240: everything cur_rand produces, plus the column/row ID parts. */
rlra_status rlra_cur_rand(rlra_ctx* ctx, int loc, const double* a, int m, int n, int64_t lda,
                          int k, int p, int q, int s, const rlra_omega* omega, int* jc, int* jr,
                          double* v, int64_t ldv, double* w, int64_t ldw, double* c,
                          int64_t ldc, double* u, int64_t ldu, double* r, int64_t ldr,
                          double* residual, double* qr_residual);

#ifdef __cplusplus
}
#endif
#endif /* RLRA_C_H */
