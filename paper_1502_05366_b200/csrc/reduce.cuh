// reduce.cuh — deterministic reductions and small data-movement kernels.
//
// Every reduction has a fixed association order (per-thread strided partial,
// warp butterfly, fixed block tree, fixed order over blocks), so results are
// bit-identical run to run — the engine's stand-in for the reference's
// thread-count-independent determinism (core/matmul.hpp:13-15,
// tests/test_matmul.cpp:73).  No floating-point atomics anywhere.
#pragma once

#include "common.cuh"

namespace rlra_b200 {

// out[0] = sum of x[0..n) in a fixed order (one CTA).
void sum_fixed_order(Context& ctx, const double* x, int64_t n, double* out);

// out[0] = sum_{i,j} A(i,j)^2 over an m x n view (fixed order); the
// Frobenius norm is its square root (reference core/norms.hpp:29-31).
void sum_squares(Context& ctx, const DMat& a, double* out_sq);

// Y = X (same shape), strided copies.
void copy_mat(Context& ctx, const DMat& src, const DMat& dst);
// dst = src^T  (src r x c, dst c x r)
void transpose_mat(Context& ctx, const DMat& src, const DMat& dst);
// dst = 0
void zero_mat(Context& ctx, const DMat& dst);
// dst = identity (first min(r,c) diagonal ones)
void eye_mat(Context& ctx, const DMat& dst);
// dst(:, j) = src(:, idx[j]), j < count
void gather_cols(Context& ctx, const DMat& src, const int* idx, int count, const DMat& dst);
// dst(i, :) = src(idx[i], :), i < count
void gather_rows(Context& ctx, const DMat& src, const int* idx, int count, const DMat& dst);
// Y = Y - X (elementwise)
void sub_inplace(Context& ctx, const DMat& y, const DMat& x);
// copy the strict upper triangle onto the lower one (square)
void symmetrize_upper(Context& ctx, const DMat& a);

// host <-> device matrix copies honouring both leading dimensions
void h2d_mat(Context& ctx, const double* h, int64_t ldh, const DMat& d);
void d2h_mat(Context& ctx, const DMat& d, double* h, int64_t ldh);

}  // namespace rlra_b200
