// qr.cuh — tall-skinny orthonormalization and QR (K3/K4 of SURVEY.md §2.2).
//
// orth / compact_qr (reference core/qr.hpp:95-129) produce the unique Q with
// diag(R) >= 0.  The fast path is CholQR2: Gram on the DMMA GEMM, blocked
// Cholesky + triangular inverse, Q = Y R^{-1} on the DMMA GEMM, twice.  It is
// exact in exact arithmetic for full column rank; when the Cholesky pivots
// reveal near rank deficiency (pivot / original diagonal < floor) the call
// falls back to a device Householder QR that restates the reference's
// reflector rules (zero-column floor 1e-300, beta = 0, propagated unit
// vector, sign fix) — the reference's own tests feed exactly-rank-deficient
// and zero-column inputs (test_qr.cpp:74-83, test_rsvd.cpp:94-100).
#pragma once

#include "common.cuh"

namespace rlra_b200 {

struct QrResult {
    bool degenerate = false;   // Householder hit a numerically zero column
    bool used_householder = false;
};

// In place: Y (m x n, m >= n) <- Q.  If R is non-null it receives the n x n
// upper-triangular factor (diag >= 0, strictly lower part zeroed).
QrResult orth_inplace(Context& ctx, const DMat& Y, const DMat* R);

// Re-orthonormalisation inside a power iteration, where only range(Y)
// feeds the next product (sketch.hpp:53-58, qb.hpp:122-125): one CholQR pass,
// span-exact; falls back to orth_inplace when the Gram is too ill-conditioned.
// The basis handed to any consumer that needs orthonormality (the final Q,
// the Q_i appended by QB) always comes from orth_inplace.
QrResult orth_span_inplace(Context& ctx, const DMat& Y);

// One CholQR pass of Y written into `out` (same shape, no aliasing) without
// the copy back; false (out untouched) when the Gram is too ill-conditioned
// for a single pass — the caller then orthonormalises Y in place.
bool orth_span_into(Context& ctx, const DMat& Y, const DMat& out);

// R^{-1} of one CholQR pass of Y (G = Y^T Y, Cholesky): false when a pivot
// falls below floor times its original diagonal (the caller then takes the
// orth_span_inplace path).
bool span_rinv(Context& ctx, const DMat& Y, const DMat& Rinv, double floor);

// Always the Householder path (used for the fallback and for tests).
QrResult householder_qr(Context& ctx, const DMat& Y, const DMat* R);

// Q (m x r) = H_0 ... H_{r-1} [I_r; 0] from reflector columns V (m x r) and
// scalars beta (device), reference core/qr.hpp:82-89.
void form_q(Context& ctx, const double* V, int64_t ldv, const double* beta, int m, int r,
            const DMat& Q);

// Upper Cholesky of a symmetric positive-definite G (n x n, upper triangle
// read) in place: G <- R (upper, lower zeroed), Rinv <- R^{-1}.  Returns false
// when a pivot fell below floor * original diagonal (or was not positive).
// dflag (device int, zeroed by the caller): OR the breakdown into it and
// return true without a host synchronisation; the caller reads it later.
bool chol_upper_inv(Context& ctx, const DMat& G, const DMat& Rinv, double floor, int* dflag = nullptr);

// G(i, i) += s
void add_diag(Context& ctx, const DMat& G, double s);

}  // namespace rlra_b200
