// dist.cuh — row-sharded multi-GPU path (dist.cu): NCCL communicator and the
// row-sharded rsvd_v2 driver.
#pragma once

#include "common.cuh"
#include "engine.cuh"

namespace rlra_b200 {

struct Comm {
    void* handle = nullptr;  // ncclComm_t
    int nranks = 1, rank = 0, device = 0;
};

void comm_unique_id(unsigned char out[128]);
void comm_init(Context& ctx, Comm& cm, const unsigned char id[128], int nranks, int rank);
void comm_destroy(Comm& cm);

// rsvd_v2 on the row block A_g (m_g x n) of an m_total x n matrix held by the
// ranks of cm; U_g (m_g x k) row-sharded like A, sigma (device, k) and V
// (n x k) replicated on every rank.
void rsvd_v2_rowsharded(Context& ctx, Comm& cm, const DMat& A, int64_t m_total, int k, int p, int q, int s,
                        OmegaSource& om, const DMat& U, double* sigma, const DMat& V, const DMat* sketched = nullptr);

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
