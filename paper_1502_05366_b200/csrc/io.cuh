// io.cuh — binary matrix I/O to device shards, the test-matrix generator and
// the SVD verifier (io.cu; reference io.hpp, testmat.hpp, report.hpp).
#pragma once

#include <string>
#include <vector>

#include "common.cuh"
#include "engine.cuh"

namespace rlra_b200 {

struct BinaryHeader {
    int rows = 0, cols = 0;
};

// io.hpp:66-109 validation (sizes, dimensions) with the reference's messages
BinaryHeader read_binary_header(const std::string& path);
// rows [row0, row0 + dst.rows) of the file into the column-major device dst
// (dst.cols == file cols); non-finite values raise RLRA_EIO
void load_binary_rows(Context& ctx, const std::string& path, int64_t row0, const DMat& dst);
// io.hpp:50-58 format from a device matrix
void save_binary(Context& ctx, const std::string& path, const DMat& src);

// testmat.hpp:65-74 semantics: A = U diag(sigma) V^T (+ noise * G), U, V the
// orthonormalised Philox Gaussian draws 101/102 of `seed`, G draw 103
void gen_test_matrix(Context& ctx, const std::vector<double>& sigma, uint64_t seed, double noise, const DMat& A);

struct VerifyReport {
    double rel_frobenius_error = 0.0;
    double rel_spectral_error = 0.0;
    double fro_floor = NAN, spec_floor = NAN, spec_bound = NAN;
};
// report.hpp:97-138 verify_reconstruction for recon = X Y^T (X m x k, Y n x k)
VerifyReport verify_lowrank(Context& ctx, const DMat& A, const DMat& X, const DMat& Y, int k,
                            const std::vector<double>& sigma_true);
// report.hpp:142-154 verify(a, SvdFactors, sigma_true); sigma on the device
VerifyReport verify_svd(Context& ctx, const DMat& A, const DMat& U, const double* sigma, const DMat& V, int k,
                        const std::vector<double>& sigma_true);

// qb.hpp:43-95 qb_single: Q (m x max_rank), B (max_rank x n, ld >= max_rank)
QbOut qb_single(Context& ctx, const DMat& A, double tol, int max_rank, OmegaSource& om, const DMat& Q,
                const DMat& B);

}  // namespace rlra_b200
