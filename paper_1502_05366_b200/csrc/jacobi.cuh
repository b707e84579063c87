// jacobi.cuh — small dense SVD / symmetric eigensolver (K5/K6 of SURVEY.md §2.2).
//
// small_svd restates reference core/jacobi.hpp:145-232: one-sided (Hestenes)
// Jacobi with the same rotation formula, the same skip rule
// |a_pq| <= 1e-15 sqrt(a_pp a_qq) (or a zero column), the same stopping rule
// (a sweep without rotations) and the same 60-sweep cap, stable descending
// sort and orthonormal completion for sigma <= 1e-300 (:33-60).  The pair
// order is the parallel round-robin tournament instead of the serial cyclic
// order, so every round's n/2 rotations run concurrently (one warp per pair)
// inside one cooperative kernel.
#pragma once

#include "common.cuh"

namespace rlra_b200 {

// A (m x n, m >= n) -> U (m x n), sigma (n, device), V (n x n).  A is not
// modified.  Throws ConvergenceError after 60 sweeps.
// upper_tri: A is square upper triangular (the R-hat of finish_qr_bt); the
// streaming kernel may then recover V as A^{-1} W (verified, jacobi.cu).
void small_svd_tall(Context& ctx, const DMat& A, const DMat& U, double* sigma, const DMat& V,
                    bool upper_tri = false);

// Raises the convergence errors small_svd_tall deferred to the end of the
// API call (ctx.svd_pending); called by the C-ABI after every entry point.
void small_svd_deferred_checks(Context& ctx);

// Any shape: r = min(m,n); U (m x r), V (n x r) (jacobi.hpp:148-152).
void small_svd(Context& ctx, const DMat& A, const DMat& U, double* sigma, const DMat& V);

// Symmetric eigendecomposition by cyclic two-sided Jacobi (jacobi.hpp:68-139):
// values descending (device), vectors n x n.
void sym_eig(Context& ctx, const DMat& T, double* values, const DMat& vectors);

}  // namespace rlra_b200
