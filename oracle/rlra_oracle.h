/*
 * rlra_oracle.h — CPU restatement of the reference's randomized low-rank
 * factorization path (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity checker, never the product: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  Every function restates the reference algorithm in plain C99
 * with the same loop and summation order, so that compiled with the same
 * flags as the reference (-O2 -ffp-contract=off) it is bit-identical to it.
 * That claim is pinned by tests/test_oracle_pin.py against oracle/_ref
 * (the unmodified reference headers compiled by oracle/Makefile) and against
 * the committed golden vectors in tests/golden/.
 *
 * Layout contract (reference core/matrix.hpp:17-80): column-major doubles,
 * element (i,j) at p[i + j*rows], leading dimension == rows.
 *
 * Status codes mirror include/rlra_c.h: 0 ok, 1 dimension, 2 numerical,
 * 3 convergence.  The message of the last failure is in orc_last_error().
 */
#ifndef RLRA_ORACLE_H
#define RLRA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint64_t s[4];
    double spare;
    int have_spare;
} orc_rng;

const char* orc_last_error(void);

/* core/rng.hpp:18-88 */
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next_u64(orc_rng* r);
double orc_rng_gaussian(orc_rng* r);
void orc_rng_substream(orc_rng* parent, orc_rng* child);
void orc_gaussian_matrix(int rows, int cols, orc_rng* r, double* out);

/* core/matmul.hpp:16-95: c (m x n) = op(a) * op(b); c is overwritten. */
int orc_matmul(int ta, int tb, const double* a, int ar, int ac, const double* b, int br, int bc,
               double* c);

/* core/norms.hpp:14-31 */
double orc_sum_squares(const double* p, int64_t n);
double orc_frobenius(const double* a, int64_t count);

/* core/qr.hpp:95-129 */
int orc_compact_qr(const double* a, int m, int n, double* q, double* r, int* degenerate);

/* core/qr.hpp:140-236.  q1 is m x kmax, s1 is kmax x n (ld = kmax) where
 * kmax = k (rank mode) or min(m,n) (tol mode); only the first frank
 * columns/rows are meaningful.  perm has n entries. */
int orc_pivoted_qr(const double* a, int m, int n, int k, double tol, double* q1, double* s1,
                   int ld_s1, int* perm, int* frank, double* residual, int* reached,
                   int* degenerate);

/* core/qr.hpp:242-275 */
int orc_upper_tri_solve(const double* s11, int lds11, int k, const double* s12, int lds12, int nc,
                        double* t, int* clamped);

/* core/jacobi.hpp:145-232: r = min(m,n); u m x r, sigma r, v n x r. */
int orc_small_svd(const double* a, int m, int n, double* u, double* sigma, double* v);

/* core/jacobi.hpp:68-139 */
int orc_sym_eig(const double* t, int n, double* values, double* vectors);

/* sketch.hpp:44-67.  sample_right -> y m x l; sample_left -> y l x n. */
int orc_sample_right(const double* a, int m, int n, int l, int q, int s, orc_rng* r, double* y);
int orc_sample_left(const double* a, int m, int n, int l, int q, int s, orc_rng* r, double* y);

/* rsvd.hpp:127-160.  variant: 0 = v2 (QR of B^T), 1 = v1 (B B^T), 2 = basic.
 * u m x k, sigma k, v n x k. */
int orc_rsvd(int variant, const double* a, int m, int n, int k, int p, int q, int s, orc_rng* r,
             double* u, double* sigma, double* v);

/* qb.hpp:98-152.  w (m x n) is destroyed and left as A - QB when inplace.
 * q has capacity m x cap, b is cap x n with ld = cap, cap >= min(b*M, min(m,n)).
 * hist has room for num_blocks entries. */
int orc_qb_blocked(const double* a, int m, int n, int blk, int num_blocks, double tol, int q_power,
                   int reorth_period, orc_rng* r, double* q, double* b, int cap, int* ell,
                   double* hist, int* nhist, double* final_resid, int* reached, double* w_out);

/* qb.hpp:276-288 + rsvd.hpp:115-160.  b has ld = ldb.  vnum 0 = QR, 1 = BBt.
 * k == 0 keeps all ell.  u m x k, sigma k, v n x k. */
int orc_svd_from_qb(const double* q, const double* b, int ldb, int m, int n, int ell, int k,
                    int vnum, double* u, double* sigma, double* v, int* k_out);

/* interp.hpp:101-117 (id_column; rank or tolerance mode).  v is n x kcap. */
int orc_id_column(const double* a, int m, int n, int k, double tol, int* jc, double* v,
                  int* k_out, double* qr_residual, int* reached, int* clamped);

/* interp.hpp:203-223 */
int orc_id_rand(const double* a, int m, int n, int k, int p, int q, int s, orc_rng* r, int* jc,
                double* v, double* qr_residual, int* clamped);

/* interp.hpp:123-140: row side of a finished column ID.  jr m, w m x k. */
int orc_two_sided_from_column(const double* a, int m, int n, const int* jc, int k, int* jr,
                              double* w);

/* interp.hpp:143-177: c m x k, u k x k, r k x n. */
int orc_cur_from_two_sided(const double* a, int m, int n, const int* jc, const int* jr,
                           const double* v, int k, double* c, double* u, double* r,
                           double* residual);

/* interp.hpp:240-244 */
int orc_cur_rand(const double* a, int m, int n, int k, int p, int q, int s, orc_rng* rng, int* jc,
                 int* jr, double* v, double* w, double* c, double* u, double* r,
                 double* residual, double* qr_residual);

/* interp.hpp:228-236 */
int orc_id_from_qb(const double* b, int ldb, int ell, int n, int k, int* jc, double* v,
                   double* qr_residual, int* clamped);

#ifdef __cplusplus
}
#endif
#endif
