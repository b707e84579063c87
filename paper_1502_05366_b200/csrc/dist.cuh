// dist.cuh — row-sharded multi-GPU path (dist.cu): NCCL communicator and the
// row-sharded rsvd_v2 driver.
#pragma once

#include <vector>

#include "common.cuh"
#include "engine.cuh"

namespace rlra_b200 {

// Host-staged collectives (rlra_host_collectives in rlra_c.h): the device
// buffer is copied to pinned host memory after the context stream drains,
// combined by the caller's functions, and copied back.  No kernel of one rank
// ever waits on another rank's kernel, so ranks may share a GPU (tests), with
// gpu_acquire/gpu_release (optional) keeping at most one rank's GPU work in
// flight at a time.
struct HostCollectives {
    int (*allreduce_sum)(void* user, double* buf, size_t count) = nullptr;
    int (*allgather)(void* user, const double* send, double* recv, size_t count) = nullptr;
    void (*gpu_acquire)(void* user) = nullptr;
    void (*gpu_release)(void* user) = nullptr;
    void* user = nullptr;
};

struct Comm {
    enum Kind { NCCL = 0, HOST = 1 };
    Kind kind = NCCL;
    void* handle = nullptr;  // ncclComm_t (NCCL)
    int nranks = 1, rank = 0, device = 0;
    HostCollectives host;     // HOST
    double* stage = nullptr;  // pinned staging (HOST), stage_cap doubles
    size_t stage_cap = 0;
    double timeout_s = 600.0;  // collective wait limit (RLRA_COMM_TIMEOUT_S)
};

void comm_unique_id(unsigned char out[128]);
void comm_init(Context& ctx, Comm& cm, const unsigned char id[128], int nranks, int rank);
void comm_init_host(Context& ctx, Comm& cm, int nranks, int rank, const HostCollectives& hc);
void comm_destroy(Comm& cm);

// Wait for the context stream with the communicator's failure detection: NCCL
// async errors are polled (ncclCommGetAsyncError) and the communicator is
// aborted (ncclCommAbort) on an error or after timeout_s, raising RLRA_ENCCL
// instead of hanging.
void comm_sync(Context& ctx, Comm& cm);

// The GPU token of a HOST communicator (no-ops otherwise): held by a rank
// while its GPU work is in flight; the rowsharded entry points take it for
// the whole call and the host collectives hand it over while they exchange.
struct CommGpuScope {
    Comm& cm;
    explicit CommGpuScope(Comm& c) : cm(c) {
        if (cm.kind == Comm::HOST && cm.host.gpu_acquire) cm.host.gpu_acquire(cm.host.user);
    }
    ~CommGpuScope() {
        if (cm.kind == Comm::HOST && cm.host.gpu_release) cm.host.gpu_release(cm.host.user);
    }
    CommGpuScope(const CommGpuScope&) = delete;
    CommGpuScope& operator=(const CommGpuScope&) = delete;
};

// An in-process group of ranks run as threads (one rlra_ctx each, any
// devices): the HostCollectives above over shared memory, with a barrier
// that times out instead of hanging.  Sums are formed in rank order on every
// rank, so every rank gets the same bits.
struct LocalGroup;
LocalGroup* local_group_create(int nranks, double timeout_s);
void local_group_destroy(LocalGroup* g);
HostCollectives local_group_collectives(LocalGroup* g, int rank);

// orthonormalise the row-sharded Y (m_g x n of an m_total x n matrix) in
// place: CholQR2 (span_only: one pass) with allreduced Grams, shifted CholQR3
// when the Gram is too ill-conditioned, TSQR (allgathered R factors) when the
// sketch is exactly rank deficient.  Every decision depends only on
// allreduced data, so all ranks take the same branch.
void orth_rowsharded(Context& ctx, Comm& cm, const DMat& Y, int64_t m_total, bool span_only);

// rows [row0, row0 + A.rows) of the test matrix gen_test_matrix (io.cuh)
// builds: U's rows are the same Philox draws (counter = global row) and are
// orthonormalised across the ranks, V is replicated; equal to the single-GPU
// generator's rows up to rounding.
void gen_test_matrix_rowsharded(Context& ctx, Comm& cm, const std::vector<double>& sigma, uint64_t seed,
                                double noise, int64_t row0, int64_t m_total, const DMat& A);

// rsvd_v2 on the row block A_g (m_g x n) of an m_total x n matrix held by the
// ranks of cm; U_g (m_g x k) row-sharded like A, sigma (device, k) and V
// (n x k) replicated on every rank.
// sketched: Y_g = A_g Omega already formed; zpre: A_g^T Y_g summed under the
// upload (the first power step then needs no pass over A_g).
void rsvd_v2_rowsharded(Context& ctx, Comm& cm, const DMat& A, int64_t m_total, int k, int p, int q, int s,
                        OmegaSource& om, const DMat& U, double* sigma, const DMat& V, const DMat* sketched = nullptr,
                        const DMat* zpre = nullptr);

// id_rand (interp.hpp:203-223) on the row-sharded A: jc (device, n) and V
// (n x k) replicated.  Omega~ is m_total x l, this rank using rows
// [row0, row0 + m_g).
IdOut id_rand_rowsharded(Context& ctx, Comm& cm, const DMat& A, int64_t row0, int64_t m_total, int k, int p,
                         int q, int s, OmegaSource& om, int* jc, const DMat& V);

// cur_rand (interp.hpp:240-244) on the row-sharded A: the column ID as above,
// the row ID of C = A(:, Jc) by a column-pivoted QR whose pivot statistics
// are allgathered every step, R = A(Jr, :) assembled by allreduce, the
// linkage replicated.  jc, V, jr (global rows), U, R replicated; W_g and C_g
// this rank's rows.  Returns ||A - C U R||_F.
double cur_rand_rowsharded(Context& ctx, Comm& cm, const DMat& A, int64_t row0, int64_t m_total, int k, int p,
                           int q, int s, OmegaSource& om, int* jc, const DMat& V, int* jr, const DMat& Wg,
                           const DMat& Cg, const DMat& U, const DMat& R, IdOut* id_out);

// qb_blocked (qb.hpp:98-142) on the row-sharded W (destroyed: left as the
// residual rows): Q (m_g x cap) row-sharded, B (cap x n) replicated.  The
// exchanges: the b x b CholQR Grams, n x b power partials, the l x b
// re-orthogonalisation projection, the b x n block B_i, and ||W||^2.
// svd_from_qb on (Q_g, B) then gives U_g, sigma, V (the lift is local).
QbOut qb_blocked_rowsharded(Context& ctx, Comm& cm, const DMat& W, int64_t m_total, int blk, int num_blocks,
                            double tol, int q_power, int reorth_period, OmegaSource& om, const DMat& Q,
                            const DMat& B);

// qb_hierarchical (qb.hpp:211-271) with num_row_blocks = world * L slabs,
// rank g holding slabs [g L, (g+1) L) (the reference's slab partition:
// floor(m_total / nrb) rows each, the last slab taking the remainder).
// Q (m_g x b*M) this rank's rows, B replicated; returns ||A - QB||_F.
double qb_hierarchical_rowsharded(Context& ctx, Comm& cm, const DMat& A, int64_t m_total, int num_row_blocks, int blk,
                                  int num_blocks, int q_power, OmegaSource& om, const DMat& Q, const DMat& B);

}  // namespace rlra_b200
