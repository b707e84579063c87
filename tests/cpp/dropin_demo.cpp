// A reference-style program (uses only the rlra:: API of the reference
// headers) compiled against include/rlra and linked with librlra_b200.so:
// the drop-in switch is the include path and the library.  Exits non-zero on
// any failed check; prints one summary line.
#include <cmath>
#include <cstdio>
#include <vector>

#include "rlra/interp.hpp"
#include "rlra/io.hpp"
#include "rlra/qb.hpp"
#include "rlra/report.hpp"
#include "rlra/rsvd.hpp"
#include "rlra/testmat.hpp"

int main(int argc, char** argv) {
    const char* tmp = argc > 1 ? argv[1] : "dropin.bin";
    rlra::RngState rng(12345);
    std::vector<double> ex(400);
    for (int j = 0; j < 400; ++j) ex[std::size_t(j)] = -j / 10.0;  // sigma_j = 10^(-j/10)
    rlra::TestMatrix t = rlra::gen_test_matrix(600, 400, rlra::SpectrumSpec::custom(ex), rng);
    rlra::save_binary(tmp, t.a);
    rlra::DenseMatrix a = rlra::load_binary(tmp);
    if (rlra::max_abs_diff(a, t.a) != 0.0) return 2;
    rlra::SvdFactors f = rlra::rsvd_v2(a, 40, 10, 2, 1, rng);
    rlra::ErrorReport e = rlra::verify(a, f, t.sigma_true);
    double worst = 0.0;
    for (int j = 0; j < 20; ++j) worst = std::fmax(worst, std::fabs(f.sigma[j] - t.sigma_true[j]) / t.sigma_true[j]);
    if (worst > 1e-8 || e.rel_frobenius_error > 10.0 * e.fro_floor + 1e-12) return 3;
    rlra::CurFactors c = rlra::cur_rand(a, 30, 10, 2, 1, rng);
    rlra::QbFactors qb = rlra::qb_blocked(a, 20, 10, 1e-3, 1, 1, rng);
    rlra::QbFactors qh = rlra::qb_hierarchical(a, 4, 10, 3, 1, rng);
    rlra::QbFactors qp = rlra::qb_parallel(a, 10, 3, 1, rng);
    if (qh.ell != 30 || qp.ell != 30 || !(qh.residual_report.final_residual > 0.0)) return 5;
    try {
        rlra::matmul(rlra::DenseMatrix(3, 4), rlra::DenseMatrix(5, 2));
        return 4;
    } catch (const rlra::DimensionError& err) {  // the reference's exception class
    }
    std::printf("dropin ok: sigma_rel %.2e rel_fro %.3e floor %.3e cur_residual %.3e qb_ell %d\n", worst,
                e.rel_frobenius_error, e.fro_floor, c.residual, qb.ell);
    return 0;
}
