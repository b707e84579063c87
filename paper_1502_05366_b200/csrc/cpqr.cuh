// cpqr.cuh — column-pivoted QR and triangular solve (K8/K9 of SURVEY.md §2.2).
#pragma once

#include "common.cuh"

namespace rlra_b200 {

struct CpqrResult {
    int frank = 0;
    double residual = 0.0;
    bool reached = false;
    bool degenerate = false;
};

// Partial column-pivoted QR restating reference core/qr.hpp:140-236:
// Businger-Golub greedy pivot on downdated squared norms with strict '>' from
// the current position (earliest position wins a tie), norm recomputation when
// a downdated value falls below 1e-6 of its reference, Householder steps with
// the reference reflector rules, sign fix diag(S11) >= 0.
//   A  (m x n) input (not modified);
//   Q1 (m x kmax) optional (q1 of the reference), may be null;
//   S1 (kmax x n) output rows [0, frank);
//   perm (device, n ints).
CpqrResult pivoted_qr(Context& ctx, const DMat& A, int k, double tol, const DMat* Q1, const DMat& S1,
                      int* perm);

// T (k x nc) = S11^{-1} S12 with the reference clamp (core/qr.hpp:242-275).
// Throws NumericalError on a zero diagonal.  Returns `clamped`.
bool upper_tri_solve(Context& ctx, const DMat& S11, const DMat& S12, const DMat& T);

// T (k x nc) <- S11^{-1} T for upper-triangular S11, blocked on DMMA (no
// clamp, no diagonal check: a zero pivot leaves inf/NaN in T).
// fast: diagonal blocks by trisolve_reg_kernel (registers + reciprocal pivots).
void upper_tri_solve_inplace(Context& ctx, const DMat& S11, const DMat& T, bool fast = false);

}  // namespace rlra_b200
