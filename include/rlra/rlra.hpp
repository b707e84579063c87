// rlra/rlra.hpp — drop-in C++ API for the B200 engine.
//
// Re-declares the reference's public API (namespace rlra, reference
// proj/include/rlra/*.hpp) with the same names, signatures, value types and
// exception classes, and implements every numerical entry point by calling
// the C-ABI in rlra_c.h, i.e. on the GPU.  A program written against the
// reference switches by putting this include directory first and linking
// librlra_b200.so.  Per-file forwarding headers (rlra/rsvd.hpp,
// rlra/core/qr.hpp, ...) exist so the reference's include lines keep working.
//
// Host-side pieces kept on the host exactly as the reference has them: the
// DenseMatrix/Permutation value types and their copy helpers, and RngState
// (the Omega stream is the reference's, drawn on the host and uploaded:
// parity mode, rlra_c.h RLRA_OMEGA_CALLBACK).
//
// Context: each host thread lazily opens one engine context on device
// $RLRA_DEVICE (default 0).  config::set_threads is accepted and ignored
// for the GPU path (it only sized the reference's CPU matmul fan-out).
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <initializer_list>
#include <numeric>
#include <stdexcept>
#include <limits>
#include <string>
#include <utility>
#include <vector>

#include "../rlra_c.h"

namespace rlra {

// ------------------------------------------------------------- errors ---
// reference core/errors.hpp:11-33
struct Error : std::runtime_error {
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};
struct DimensionError : Error {
    using Error::Error;
};
struct NumericalError : Error {
    using Error::Error;
};
struct ConvergenceError : Error {
    using Error::Error;
};
struct IoError : Error {
    using Error::Error;
};

namespace detail {
inline std::string msg(const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    return buf;
}

[[noreturn]] inline void throw_status(rlra_status st) {
    const std::string m = rlra_last_error();
    switch (st) {
        case RLRA_EDIM: throw DimensionError(m);
        case RLRA_ENUM: throw NumericalError(m);
        case RLRA_ECONV: throw ConvergenceError(m);
        case RLRA_EIO: throw IoError(m);
        default: throw Error(m);
    }
}
inline void check(rlra_status st) {
    if (st != RLRA_OK) throw_status(st);
}

struct CtxHolder {
    rlra_ctx* ctx = nullptr;
    ~CtxHolder() {
        if (ctx) rlra_ctx_destroy(ctx);
    }
};
inline rlra_ctx* ctx() {
    thread_local CtxHolder h;
    if (!h.ctx) {
        const char* d = std::getenv("RLRA_DEVICE");
        check(rlra_ctx_create(d ? std::atoi(d) : 0, &h.ctx));
    }
    return h.ctx;
}
}  // namespace detail

// ------------------------------------------------------------- config ---
namespace config {
inline std::atomic<int>& thread_count_ref() {
    static std::atomic<int> n{1};
    return n;
}
inline void set_threads(int n) { thread_count_ref().store(std::max(1, n)); }
inline int threads() { return thread_count_ref().load(); }
}  // namespace config

// ------------------------------------------------------- value types ---
// Column-major doubles, element (i,j) at data()[i + j*rows()]
// (reference core/matrix.hpp:17-80).
class DenseMatrix {
public:
    DenseMatrix() = default;
    DenseMatrix(int rows, int cols) : r_(rows), c_(cols) {
        if (rows < 0 || cols < 0)
            throw DimensionError(detail::msg("DenseMatrix: negative dimensions %dx%d", rows, cols));
        v_.assign(std::size_t(rows) * std::size_t(cols), 0.0);
    }
    DenseMatrix(std::initializer_list<std::initializer_list<double>> rows_list) {
        r_ = int(rows_list.size());
        c_ = r_ ? int(rows_list.begin()->size()) : 0;
        v_.assign(std::size_t(r_) * c_, 0.0);
        int i = 0;
        for (const auto& row : rows_list) {
            if (int(row.size()) != c_) throw DimensionError("DenseMatrix: ragged initializer list");
            int j = 0;
            for (double x : row) (*this)(i, j++) = x;
            ++i;
        }
    }
    static DenseMatrix identity(int n) {
        DenseMatrix e(n, n);
        for (int i = 0; i < n; ++i) e(i, i) = 1.0;
        return e;
    }
    static DenseMatrix diag(const std::vector<double>& d) {
        DenseMatrix e(int(d.size()), int(d.size()));
        for (int i = 0; i < int(d.size()); ++i) e(i, i) = d[i];
        return e;
    }
    int rows() const { return r_; }
    int cols() const { return c_; }
    std::size_t size() const { return v_.size(); }
    double& operator()(int i, int j) { return v_[std::size_t(i) + std::size_t(j) * r_]; }
    double operator()(int i, int j) const { return v_[std::size_t(i) + std::size_t(j) * r_]; }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    double* col(int j) { return v_.data() + std::size_t(j) * r_; }
    const double* col(int j) const { return v_.data() + std::size_t(j) * r_; }
    bool all_finite() const {
        return std::all_of(v_.begin(), v_.end(), [](double x) { return std::isfinite(x); });
    }

private:
    int r_ = 0, c_ = 0;
    std::vector<double> v_;
};

// 0-based bijection (core/matrix.hpp:83-110)
class Permutation {
public:
    Permutation() = default;
    explicit Permutation(std::vector<int> idx) : p_(std::move(idx)) {
        std::vector<char> seen(p_.size(), 0);
        for (int x : p_) {
            if (x < 0 || x >= int(p_.size()))
                throw DimensionError(detail::msg("Permutation: index %d out of range [0,%zu)", x, p_.size()));
            if (seen[x]) throw DimensionError(detail::msg("Permutation: duplicate index %d", x));
            seen[x] = 1;
        }
    }
    static Permutation identity(int n) {
        std::vector<int> v(n);
        std::iota(v.begin(), v.end(), 0);
        return Permutation(std::move(v));
    }
    int operator[](int i) const { return p_[std::size_t(i)]; }
    int size() const { return int(p_.size()); }
    const std::vector<int>& indices() const { return p_; }

private:
    std::vector<int> p_;
};

inline DenseMatrix transpose(const DenseMatrix& a) {
    DenseMatrix t(a.cols(), a.rows());
    for (int j = 0; j < a.cols(); ++j)
        for (int i = 0; i < a.rows(); ++i) t(j, i) = a(i, j);
    return t;
}
inline DenseMatrix submatrix(const DenseMatrix& a, int r0, int nr, int c0, int nc) {
    if (r0 < 0 || c0 < 0 || nr < 0 || nc < 0 || r0 + nr > a.rows() || c0 + nc > a.cols())
        throw DimensionError(detail::msg("submatrix: block %d+%d x %d+%d exceeds %dx%d", r0, nr, c0, nc,
                                         a.rows(), a.cols()));
    DenseMatrix b(nr, nc);
    for (int j = 0; j < nc; ++j) std::copy(a.col(c0 + j) + r0, a.col(c0 + j) + r0 + nr, b.col(j));
    return b;
}
inline DenseMatrix select_columns(const DenseMatrix& a, const Permutation& idx, int count) {
    if (count < 0 || count > idx.size() || count > a.cols())
        throw DimensionError(detail::msg("select_columns: count %d out of range", count));
    DenseMatrix c(a.rows(), count);
    for (int j = 0; j < count; ++j) std::copy(a.col(idx[j]), a.col(idx[j]) + a.rows(), c.col(j));
    return c;
}
inline DenseMatrix select_rows(const DenseMatrix& a, const Permutation& idx, int count) {
    if (count < 0 || count > idx.size() || count > a.rows())
        throw DimensionError(detail::msg("select_rows: count %d out of range", count));
    DenseMatrix r(count, a.cols());
    for (int j = 0; j < a.cols(); ++j)
        for (int i = 0; i < count; ++i) r(i, j) = a(idx[i], j);
    return r;
}
inline DenseMatrix hconcat(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.rows() != b.rows())
        throw DimensionError(detail::msg("hconcat: row counts disagree (%d vs %d)", a.rows(), b.rows()));
    DenseMatrix c(a.rows(), a.cols() + b.cols());
    std::copy(a.data(), a.data() + a.size(), c.data());
    std::copy(b.data(), b.data() + b.size(), c.data() + a.size());
    return c;
}
inline DenseMatrix vconcat(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.cols() != b.cols())
        throw DimensionError(detail::msg("vconcat: column counts disagree (%d vs %d)", a.cols(), b.cols()));
    DenseMatrix c(a.rows() + b.rows(), a.cols());
    for (int j = 0; j < a.cols(); ++j) {
        std::copy(a.col(j), a.col(j) + a.rows(), c.col(j));
        std::copy(b.col(j), b.col(j) + b.rows(), c.col(j) + a.rows());
    }
    return c;
}
namespace detail {
template <class Op>
DenseMatrix zip(const DenseMatrix& a, const DenseMatrix& b, const char* name, Op op) {
    if (a.rows() != b.rows() || a.cols() != b.cols())
        throw DimensionError(msg("%s: shapes disagree (%dx%d vs %dx%d)", name, a.rows(), a.cols(), b.rows(),
                                 b.cols()));
    DenseMatrix c(a.rows(), a.cols());
    for (std::size_t i = 0; i < a.size(); ++i) c.data()[i] = op(a.data()[i], b.data()[i]);
    return c;
}
}  // namespace detail
inline DenseMatrix subtract(const DenseMatrix& a, const DenseMatrix& b) {
    return detail::zip(a, b, "subtract", [](double x, double y) { return x - y; });
}
inline DenseMatrix add(const DenseMatrix& a, const DenseMatrix& b) {
    return detail::zip(a, b, "add", [](double x, double y) { return x + y; });
}
inline DenseMatrix scale(const DenseMatrix& a, double s) {
    DenseMatrix c(a.rows(), a.cols());
    for (std::size_t i = 0; i < a.size(); ++i) c.data()[i] = s * a.data()[i];
    return c;
}
inline void scale_columns_inplace(DenseMatrix& a, const std::vector<double>& s) {
    if (int(s.size()) != a.cols())
        throw DimensionError(detail::msg("scale_columns_inplace: %zu factors for %d columns", s.size(), a.cols()));
    for (int j = 0; j < a.cols(); ++j)
        for (int i = 0; i < a.rows(); ++i) a(i, j) *= s[j];
}
inline double max_abs_diff(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols()) throw DimensionError("max_abs_diff: shapes disagree");
    double m = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a.data()[i] - b.data()[i]));
    return m;
}

// ---------------------------------------------------------------- rng ---
// The reference stream (core/rng.hpp:18-87) through the library's host RNG.
class RngState {
public:
    explicit RngState(std::uint64_t seed = 0) { rlra_rng_seed(&s_, seed); }
    std::uint64_t next_u64() { return rlra_rng_next_u64(&s_); }
    double next_unit() { return double(next_u64() >> 11) * 0x1.0p-53; }
    double next_gaussian() { return rlra_rng_next_gaussian(&s_); }
    RngState substream() {
        RngState c;
        rlra_rng_substream(&s_, &c.s_);
        return c;
    }
    rlra_rng* raw() { return &s_; }

private:
    rlra_rng s_{};
};

inline DenseMatrix gaussian_matrix(int rows, int cols, RngState& rng) {
    DenseMatrix g(rows, cols);
    rlra_rng_gaussian_fill(rng.raw(), rows, cols, g.data());
    return g;
}

namespace detail {
inline rlra_omega omega_from(RngState& rng, bool substreams) {
    rlra_omega o{};
    o.mode = RLRA_OMEGA_CALLBACK;
    o.fill = substreams ? rlra_omega_fill_rng_substream : rlra_omega_fill_rng;
    o.user = rng.raw();
    return o;
}
inline int ld(const DenseMatrix& a) { return std::max(1, a.rows()); }
}  // namespace detail

// ------------------------------------------------------------ kernels ---
inline DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b, bool trans_a = false,
                          bool trans_b = false) {
    const int m = trans_a ? a.cols() : a.rows(), n = trans_b ? b.rows() : b.cols();
    const int ka = trans_a ? a.rows() : a.cols(), kb = trans_b ? b.cols() : b.rows();
    if (ka != kb)
        throw DimensionError(detail::msg("matmul: inner dimensions disagree: op(%dx%d) * op(%dx%d)", a.rows(),
                                         a.cols(), b.rows(), b.cols()));
    DenseMatrix c(m, n);
    if (m == 0 || n == 0) return c;
    detail::check(rlra_matmul(detail::ctx(), RLRA_HOST, trans_a, trans_b, a.data(), a.rows(), a.cols(),
                              detail::ld(a), b.data(), b.rows(), b.cols(), detail::ld(b), c.data(),
                              std::max(1, m)));
    return c;
}

inline double frobenius_norm(const DenseMatrix& a) {
    if (a.size() == 0) return 0.0;
    double out = 0.0;
    detail::check(rlra_frobenius_norm(detail::ctx(), RLRA_HOST, a.data(), a.rows(), a.cols(), detail::ld(a), &out));
    return out;
}
inline double column_norm(const DenseMatrix& a, int j) {
    double out = 0.0;
    if (a.rows() == 0) return 0.0;
    detail::check(rlra_frobenius_norm(detail::ctx(), RLRA_HOST, a.col(j), a.rows(), 1, a.rows(), &out));
    return out;
}
inline double spectral_norm_est(const DenseMatrix& a, int iters, RngState& rng) {  // norms.hpp:41-56
    if (iters < 20) throw DimensionError(detail::msg("spectral_norm_est: iters=%d, need >= 20", iters));
    if (a.rows() == 0 || a.cols() == 0) return 0.0;
    DenseMatrix v = gaussian_matrix(a.cols(), 1, rng);
    double sigma = 0.0;
    for (int it = 0; it < iters; ++it) {
        const double vn = frobenius_norm(v);
        if (vn == 0.0) return 0.0;
        for (int i = 0; i < v.rows(); ++i) v(i, 0) /= vn;
        DenseMatrix w = matmul(a, v);
        sigma = frobenius_norm(w);
        v = matmul(a, w, true);
    }
    return sigma;
}

struct QrFactors {
    DenseMatrix q;
    DenseMatrix r;
    bool degenerate_rank = false;
};
struct PivotedQr {
    DenseMatrix q1;
    DenseMatrix s1;
    Permutation perm;
    int frank = 0;
    double residual = 0.0;
    bool tolerance_reached = false;
    bool degenerate_rank = false;
};
struct TriSolve {
    DenseMatrix t;
    bool clamped = false;
};

inline QrFactors compact_qr(const DenseMatrix& a) {
    const int m = a.rows(), n = a.cols();
    if (m < n) throw DimensionError(detail::msg("compact_qr: matrix is %dx%d, need rows >= cols", m, n));
    QrFactors f{DenseMatrix(m, n), DenseMatrix(n, n), false};
    if (n == 0) return f;
    int deg = 0;
    detail::check(rlra_compact_qr(detail::ctx(), RLRA_HOST, a.data(), m, n, detail::ld(a), f.q.data(), m,
                                  f.r.data(), n, &deg));
    f.degenerate_rank = deg != 0;
    return f;
}
inline DenseMatrix orth(const DenseMatrix& a, bool* degenerate = nullptr) {
    QrFactors f = compact_qr(a);
    if (degenerate) *degenerate = f.degenerate_rank;
    return f.q;
}
inline PivotedQr pivoted_qr_partial(const DenseMatrix& a, int k, double tol = 0.0) {
    const int m = a.rows(), n = a.cols(), rmax = std::min(m, n);
    const bool tol_mode = k == 0 && tol > 0.0;
    const int kmax = tol_mode ? rmax : std::max(k, 1);
    DenseMatrix q1(m, kmax), s1(kmax, n);
    std::vector<int> perm(n);
    int frank = 0, reached = 0, deg = 0;
    double res = 0.0;
    detail::check(rlra_pivoted_qr(detail::ctx(), RLRA_HOST, a.data(), m, n, detail::ld(a), k, tol, q1.data(),
                                  std::max(1, m), s1.data(), kmax, perm.data(), &frank, &res, &reached, &deg));
    PivotedQr out;
    out.q1 = submatrix(q1, 0, m, 0, frank);
    out.s1 = submatrix(s1, 0, frank, 0, n);
    out.perm = Permutation(std::move(perm));
    out.frank = frank;
    out.residual = res;
    out.tolerance_reached = reached != 0;
    out.degenerate_rank = deg != 0;
    return out;
}
inline TriSolve upper_tri_solve(const DenseMatrix& s11, const DenseMatrix& s12) {
    const int k = s11.rows();
    if (s11.cols() != k) throw DimensionError(detail::msg("upper_tri_solve: S11 is %dx%d, need square", k, s11.cols()));
    if (s12.rows() != k) throw DimensionError(detail::msg("upper_tri_solve: S12 has %d rows, need %d", s12.rows(), k));
    TriSolve out{DenseMatrix(k, s12.cols()), false};
    if (k == 0) return out;
    int cl = 0;
    detail::check(rlra_upper_tri_solve(detail::ctx(), RLRA_HOST, s11.data(), k, k, s12.data(), s12.cols(), k,
                                       out.t.data(), k, &cl));
    out.clamped = cl != 0;
    return out;
}

struct SymEig {
    std::vector<double> values;
    DenseMatrix vectors;
};
struct SvdFactors {
    DenseMatrix u;
    std::vector<double> sigma;
    DenseMatrix v;
    int k = 0;
};

inline SymEig sym_eig(const DenseMatrix& t) {
    const int n = t.rows();
    if (t.cols() != n) throw DimensionError(detail::msg("sym_eig: matrix is %dx%d, need square", n, t.cols()));
    SymEig e{std::vector<double>(n), DenseMatrix(n, n)};
    if (n == 0) return e;
    detail::check(rlra_sym_eig(detail::ctx(), RLRA_HOST, t.data(), n, n, e.values.data(), e.vectors.data(), n));
    return e;
}
inline SvdFactors small_svd(const DenseMatrix& a) {
    const int m = a.rows(), n = a.cols(), r = std::min(m, n);
    SvdFactors f{DenseMatrix(m, r), std::vector<double>(r), DenseMatrix(n, r), r};
    if (r == 0) return f;
    detail::check(rlra_small_svd(detail::ctx(), RLRA_HOST, a.data(), m, n, detail::ld(a), f.u.data(),
                                 std::max(1, m), f.sigma.data(), f.v.data(), std::max(1, n)));
    return f;
}

// ------------------------------------------------------------- sketch ---
enum class Vnum { kQr, kBbt };

struct SketchParams {  // sketch.hpp:18-39
    int k = 0;
    int p = 5;
    int q = 1;
    int s = 1;
    double tol = 0.0;
    int block = 20;
    int max_blocks = 12;
    Vnum vnum = Vnum::kQr;
    std::uint64_t seed = 0;
    void validate(int m, int n) const {
        if ((k >= 1) == (tol > 0.0))
            throw DimensionError(detail::msg(
                "SketchParams: exactly one of rank (k=%d) and tolerance (tol=%g) must be set", k, tol));
        if (k >= 1 && k + p > std::min(m, n))
            throw DimensionError(detail::msg("SketchParams: k+p = %d exceeds min(m,n) = %d for %dx%d", k + p,
                                             std::min(m, n), m, n));
        if (p < 0 || q < 0 || s < 1 || block < 1 || max_blocks < 1 || tol < 0.0 || k < 0)
            throw DimensionError("SketchParams: negative or zero-valued parameter out of range");
    }
};

inline DenseMatrix sample_right(const DenseMatrix& a, int l, int q, int s, RngState& rng) {
    DenseMatrix y(a.rows(), std::max(l, 0));
    rlra_omega om = detail::omega_from(rng, false);
    detail::check(rlra_sample(detail::ctx(), RLRA_HOST, 0, a.data(), a.rows(), a.cols(), detail::ld(a), l, q, s,
                              &om, y.data(), std::max(1, a.rows())));
    return y;
}
inline DenseMatrix sample_left(const DenseMatrix& a, int l, int q, int s, RngState& rng) {
    DenseMatrix y(std::max(l, 0), a.cols());
    rlra_omega om = detail::omega_from(rng, false);
    detail::check(rlra_sample(detail::ctx(), RLRA_HOST, 1, a.data(), a.rows(), a.cols(), detail::ld(a), l, q, s,
                              &om, y.data(), std::max(1, l)));
    return y;
}

// --------------------------------------------------------------- rsvd ---
namespace detail {
inline SvdFactors rsvd_call(int variant, const DenseMatrix& a, int k, int p, int q, int s, RngState& rng) {
    const int kk = std::max(k, 0);
    SvdFactors f{DenseMatrix(a.rows(), kk), std::vector<double>(kk), DenseMatrix(a.cols(), kk), kk};
    rlra_omega om = omega_from(rng, false);
    check(rlra_rsvd(ctx(), RLRA_HOST, variant, a.data(), a.rows(), a.cols(), ld(a), k, p, q, s, &om, f.u.data(),
                    std::max(1, a.rows()), f.sigma.data(), f.v.data(), std::max(1, a.cols())));
    return f;
}
inline SvdFactors truncate_svd(const SvdFactors& f, int k) {
    if (k < 0 || k > f.k) throw DimensionError(msg("truncation rank %d outside [0, %d]", k, f.k));
    SvdFactors out;
    out.k = k;
    out.u = submatrix(f.u, 0, f.u.rows(), 0, k);
    out.v = submatrix(f.v, 0, f.v.rows(), 0, k);
    out.sigma.assign(f.sigma.begin(), f.sigma.begin() + k);
    return out;
}
}  // namespace detail

inline SvdFactors svd_truncated(const DenseMatrix& a, int k, double tol = 0.0) {  // rsvd.hpp:98-123
    const int r = std::min(a.rows(), a.cols());
    const bool rank_mode = k >= 1 && tol == 0.0, tol_mode = k == 0 && tol > 0.0;
    if (!rank_mode && !tol_mode)
        throw DimensionError(detail::msg("exactly one of rank k >= 1 or tol > 0 must be set (got k=%d, tol=%g)", k, tol));
    if (rank_mode && k > r) throw DimensionError(detail::msg("rank %d exceeds min(m,n) = %d", k, r));
    if (r > 2000)
        throw DimensionError(detail::msg(
            "min(m,n) = %d exceeds the dense SVD limit of 2000; use the randomized routines for matrices this large", r));
    SvdFactors full = small_svd(a);
    int keep = k;
    if (tol_mode) {
        keep = r;
        for (int i = 0; i < r; ++i)
            if (full.sigma[i] < tol) {
                keep = i;
                break;
            }
    }
    return detail::truncate_svd(full, keep);
}
inline SvdFactors rsvd_basic(const DenseMatrix& a, int k, int p, RngState& rng) {
    return detail::rsvd_call(RLRA_RSVD_BASIC, a, k, p, 0, 1, rng);
}
inline SvdFactors rsvd_v1(const DenseMatrix& a, int k, int p, int q_power, int s, RngState& rng) {
    return detail::rsvd_call(RLRA_RSVD_V1, a, k, p, q_power, s, rng);
}
inline SvdFactors rsvd_v2(const DenseMatrix& a, int k, int p, int q_power, int s, RngState& rng) {
    return detail::rsvd_call(RLRA_RSVD_V2, a, k, p, q_power, s, rng);
}

// ----------------------------------------------------------------- qb ---
struct ResidualReport {
    double final_residual = 0.0;
    std::vector<double> history;
    bool tolerance_reached = true;
};
struct QbFactors {
    DenseMatrix q;
    DenseMatrix b;
    int ell = 0;
    ResidualReport residual_report;
};

namespace detail {
inline QbFactors qb_call(DenseMatrix& w, bool inplace, int b, int num_blocks, double tol, int q_power,
                         int reorth_period, RngState& rng) {
    const int m = w.rows(), n = w.cols();
    const int cap = (b >= 1 && num_blocks >= 1) ? std::max(1, int(std::min<long long>(
                                                              (long long)b * num_blocks, std::min(m, n))))
                                                : 1;
    DenseMatrix Q(m, cap), B(cap, n);
    std::vector<double> hist(std::max(num_blocks, 1));
    int ell = 0, nh = 0, reached = 0;
    double fin = 0.0;
    rlra_omega om = omega_from(rng, true);
    check(rlra_qb_blocked(ctx(), RLRA_HOST, w.data(), m, n, ld(w), inplace ? 1 : 0, b, num_blocks, tol, q_power,
                          reorth_period, &om, Q.data(), std::max(1, m), B.data(), cap, cap, &ell, hist.data(), &nh,
                          &fin, &reached));
    QbFactors f;
    f.q = submatrix(Q, 0, m, 0, ell);
    f.b = submatrix(B, 0, ell, 0, n);
    f.ell = ell;
    f.residual_report.history.assign(hist.begin(), hist.begin() + nh);
    f.residual_report.final_residual = fin;
    f.residual_report.tolerance_reached = reached != 0;
    return f;
}
}  // namespace detail

inline QbFactors qb_blocked_inplace(DenseMatrix& w, int b, int num_blocks, double tol, int q_power,
                                    int reorth_period, RngState& rng) {
    return detail::qb_call(w, true, b, num_blocks, tol, q_power, reorth_period, rng);
}
inline QbFactors qb_blocked(const DenseMatrix& a, int b, int num_blocks, double tol, int q_power,
                            int reorth_period, RngState& rng) {
    DenseMatrix w = a;
    return detail::qb_call(w, false, b, num_blocks, tol, q_power, reorth_period, rng);
}

namespace detail {
// the composite drivers: node streams drawn from rng in the reference's order
template <class F>
inline QbFactors qb_composite(const DenseMatrix& a, int rank, int count, bool substream_per_draw, RngState& rng,
                              F&& call) {
    std::vector<rlra_rng> nodes(static_cast<std::size_t>(count));
    for (auto& nd : nodes) rlra_rng_substream(rng.raw(), &nd);
    rlra_rng_nodes holder{nodes.data(), count, substream_per_draw ? 1 : 0};
    rlra_omega om{};
    om.mode = RLRA_OMEGA_CALLBACK;
    om.fill = rlra_omega_fill_rng_nodes;
    om.user = &holder;
    QbFactors f;
    f.q = DenseMatrix(a.rows(), rank);
    f.b = DenseMatrix(rank, a.cols());
    double fin = 0.0;
    check(call(&om, f.q.data(), f.b.data(), &fin));
    f.ell = rank;
    f.residual_report.final_residual = fin;
    f.residual_report.history.push_back(fin);
    return f;
}
}  // namespace detail

// qb.hpp:159-204: M independently sampled blocks, projected sequentially
inline QbFactors qb_parallel(const DenseMatrix& a, int b, int num_blocks, int q_power, RngState& rng) {
    const int rank = (b >= 1 && num_blocks >= 1) ? b * num_blocks : 1;
    return detail::qb_composite(a, rank, std::max(num_blocks, 1), false, rng, [&](rlra_omega* om, double* q, double* bb,
                                                                                   double* fin) {
        return rlra_qb_parallel(detail::ctx(), RLRA_HOST, a.data(), a.rows(), a.cols(), detail::ld(a), b, num_blocks,
                                q_power, om, q, std::max(1, a.rows()), bb, std::max(1, rank), fin);
    });
}

// qb.hpp:211-271: leaf QBs of 2^j row slabs merged pairwise up a binary tree
inline QbFactors qb_hierarchical(const DenseMatrix& a, int num_row_blocks, int b, int num_blocks, int q_power,
                                 RngState& rng) {
    const int rank = (b >= 1 && num_blocks >= 1) ? b * num_blocks : 1;
    const int count = std::max(1, 2 * num_row_blocks - 1);
    return detail::qb_composite(a, rank, count, true, rng, [&](rlra_omega* om, double* q, double* bb, double* fin) {
        return rlra_qb_hierarchical(detail::ctx(), RLRA_HOST, a.data(), a.rows(), a.cols(), detail::ld(a),
                                    num_row_blocks, b, num_blocks, q_power, om, q, std::max(1, a.rows()), bb,
                                    std::max(1, rank), fin);
    });
}

inline SvdFactors svd_from_qb(const QbFactors& qb, int k, Vnum vnum) {
    if (k < 0 || k > qb.ell) throw DimensionError(detail::msg("rank k = %d outside [0, rank(B) = %d]", k, qb.ell));
    const int kk = k == 0 ? qb.ell : k;
    SvdFactors f{DenseMatrix(qb.q.rows(), kk), std::vector<double>(kk), DenseMatrix(qb.b.cols(), kk), kk};
    if (kk == 0) return f;
    int ko = 0;
    detail::check(rlra_svd_from_qb(detail::ctx(), RLRA_HOST, qb.q.data(), qb.q.rows(), std::max(1, qb.q.rows()),
                                   qb.b.data(), qb.b.cols(), std::max(1, qb.b.rows()), qb.ell, k,
                                   vnum == Vnum::kBbt ? RLRA_VNUM_BBT : RLRA_VNUM_QR, f.u.data(),
                                   std::max(1, qb.q.rows()), f.sigma.data(), f.v.data(),
                                   std::max(1, qb.b.cols()), &ko));
    return f;
}

// ------------------------------------------------------------- interp ---
struct IdFactors {
    Permutation jc;
    DenseMatrix v;
    int k = 0;
    double qr_residual = 0.0;
    bool tolerance_reached = true;
    bool clamped = false;
};
struct RowIdFactors {
    Permutation jr;
    DenseMatrix w;
    int k = 0;
    double qr_residual = 0.0;
    bool tolerance_reached = true;
    bool clamped = false;
};
struct TwoSidedIdFactors {
    Permutation jr;
    Permutation jc;
    DenseMatrix w;
    DenseMatrix v;
    int k = 0;
    double qr_residual = 0.0;
    bool tolerance_reached = true;
};
struct CurFactors {
    DenseMatrix c;
    DenseMatrix u;
    DenseMatrix r;
    Permutation jr;
    Permutation jc;
    int k = 0;
    double residual = 0.0;
    double qr_residual = 0.0;
    bool tolerance_reached = true;
};

inline IdFactors id_column(const DenseMatrix& a, int k, double tol = 0.0) {
    const int m = a.rows(), n = a.cols();
    const int kcap = (k == 0 && tol > 0.0) ? std::min(m, n) : std::max(k, 1);
    std::vector<int> jc(n);
    DenseMatrix v(n, kcap);
    int ko = 0, reached = 0, cl = 0;
    double res = 0.0;
    detail::check(rlra_id_column(detail::ctx(), RLRA_HOST, a.data(), m, n, detail::ld(a), k, tol, jc.data(),
                                 v.data(), std::max(1, n), &ko, &res, &reached, &cl));
    IdFactors f;
    f.jc = Permutation(std::move(jc));
    f.v = submatrix(v, 0, n, 0, ko);
    f.k = ko;
    f.qr_residual = res;
    f.tolerance_reached = reached != 0;
    f.clamped = cl != 0;
    return f;
}
inline RowIdFactors id_row(const DenseMatrix& a, int k, double tol = 0.0) {
    IdFactors c = id_column(transpose(a), k, tol);
    return RowIdFactors{std::move(c.jc), std::move(c.v), c.k, c.qr_residual, c.tolerance_reached, c.clamped};
}

namespace detail {
inline TwoSidedIdFactors two_sided_from_column(const DenseMatrix& a, IdFactors col) {
    TwoSidedIdFactors out;
    out.jc = std::move(col.jc);
    out.v = std::move(col.v);
    out.k = col.k;
    out.qr_residual = col.qr_residual;
    out.tolerance_reached = col.tolerance_reached;
    const int m = a.rows();
    std::vector<int> jr(m);
    out.w = DenseMatrix(m, out.k);
    check(rlra_two_sided_from_column(ctx(), RLRA_HOST, a.data(), m, a.cols(), ld(a), out.jc.indices().data(),
                                     out.k, jr.data(), out.w.data(), std::max(1, m)));
    out.jr = Permutation(std::move(jr));
    return out;
}
// interp.hpp:143-156: U = argmin ||U R - V^T||_F (compact QR of R^T on the
// device); a rank-deficient R names the offending skeleton row jr[i].
inline DenseMatrix cur_linkage(const DenseMatrix& r, const DenseMatrix& v, const Permutation& jr) {
    const int k = r.rows();
    DenseMatrix u(k, k);
    if (k == 0) return u;
    if (jr.size() < k) throw DimensionError(msg("cur_linkage: %d skeleton rows for rank %d", jr.size(), k));
    if (v.rows() != r.cols() || v.cols() != k)
        throw DimensionError(msg("cur_linkage: V is %dx%d, need %dx%d", v.rows(), v.cols(), r.cols(), k));
    check(rlra_cur_linkage(ctx(), RLRA_HOST, r.data(), k, r.cols(), std::max(1, k), v.data(), std::max(1, v.rows()),
                           jr.indices().data(), u.data(), std::max(1, k)));
    return u;
}
inline CurFactors cur_from_two_sided(const DenseMatrix& a, const TwoSidedIdFactors& ts) {
    CurFactors out;
    out.k = ts.k;
    out.jc = ts.jc;
    out.jr = ts.jr;
    out.qr_residual = ts.qr_residual;
    out.tolerance_reached = ts.tolerance_reached;
    out.c = DenseMatrix(a.rows(), ts.k);
    out.u = DenseMatrix(ts.k, ts.k);
    out.r = DenseMatrix(ts.k, a.cols());
    check(rlra_cur_from_two_sided(ctx(), RLRA_HOST, a.data(), a.rows(), a.cols(), ld(a), ts.jc.indices().data(),
                                  ts.jr.indices().data(), ts.v.data(), std::max(1, ts.v.rows()), ts.k,
                                  out.c.data(), std::max(1, a.rows()), out.u.data(), std::max(1, ts.k),
                                  out.r.data(), std::max(1, ts.k), &out.residual));
    return out;
}
}  // namespace detail

inline TwoSidedIdFactors id_two_sided(const DenseMatrix& a, int k, double tol = 0.0) {
    return detail::two_sided_from_column(a, id_column(a, k, tol));
}
inline CurFactors cur(const DenseMatrix& a, int k, double tol = 0.0) {
    return detail::cur_from_two_sided(a, id_two_sided(a, k, tol));
}
inline IdFactors id_rand(const DenseMatrix& a, int k, int p, int q_power, int s, RngState& rng) {
    const int n = a.cols();
    std::vector<int> jc(n);
    DenseMatrix v(n, std::max(k, 0));
    double res = 0.0;
    int cl = 0;
    rlra_omega om = detail::omega_from(rng, false);
    detail::check(rlra_id_rand(detail::ctx(), RLRA_HOST, a.data(), a.rows(), n, detail::ld(a), k, p, q_power, s,
                               &om, jc.data(), v.data(), std::max(1, n), &res, &cl));
    IdFactors f;
    f.jc = Permutation(std::move(jc));
    f.v = std::move(v);
    f.k = k;
    f.qr_residual = res;
    f.clamped = cl != 0;
    return f;
}
inline IdFactors id_from_qb(const QbFactors& qb, const DenseMatrix& a, int k) {
    if (a.rows() != qb.q.rows() || a.cols() != qb.b.cols())
        throw DimensionError(detail::msg("id_from_qb: matrix is %dx%d but the QB factors describe %dx%d", a.rows(),
                                         a.cols(), qb.q.rows(), qb.b.cols()));
    if (k < 1 || k > qb.ell) throw DimensionError(detail::msg("rank k = %d outside [1, rank(B) = %d]", k, qb.ell));
    return id_column(qb.b, k, 0.0);
}
inline CurFactors cur_rand(const DenseMatrix& a, int k, int p, int q_power, int s, RngState& rng) {
    IdFactors col = id_rand(a, k, p, q_power, s, rng);
    return detail::cur_from_two_sided(a, detail::two_sided_from_column(a, std::move(col)));
}

// ---------------------------------------------------------------- io.hpp ---
// Binary matrix files (io.hpp:40-109): same format, validation and messages;
// the engine streams the rows through the GPU (csrc/io.cu).
inline void save_binary(const std::string& path, const DenseMatrix& a) {
    detail::check(rlra_save_binary(detail::ctx(), RLRA_HOST, path.c_str(), a.data(), a.rows(), a.cols(), detail::ld(a)));
}
inline DenseMatrix load_binary(const std::string& path) {
    int m = 0, n = 0;
    detail::check(rlra_binary_header(path.c_str(), &m, &n));
    DenseMatrix a(m, n);
    detail::check(rlra_load_binary(detail::ctx(), RLRA_HOST, path.c_str(), 0, m, a.data(), detail::ld(a)));
    return a;
}

// ----------------------------------------------------------- testmat.hpp ---
struct SpectrumSpec {  // testmat.hpp:16-53
    enum class Kind { kTypeI, kTypeII, kTypeIII, kCustom };
    Kind kind = Kind::kTypeII;
    std::vector<double> custom_exponents;
    static SpectrumSpec type_i() { return {Kind::kTypeI, {}}; }
    static SpectrumSpec type_ii() { return {Kind::kTypeII, {}}; }
    static SpectrumSpec type_iii() { return {Kind::kTypeIII, {}}; }
    static SpectrumSpec custom(std::vector<double> exponents) {
        for (std::size_t i = 0; i + 1 < exponents.size(); ++i)
            if (exponents[i] < exponents[i + 1])
                throw DimensionError("SpectrumSpec: custom exponents must be nonincreasing");
        return {Kind::kCustom, std::move(exponents)};
    }
    std::vector<double> sigma(int r) const {
        if (r < 1) throw DimensionError("SpectrumSpec: rank must be positive");
        std::vector<double> exps;
        if (kind == Kind::kCustom) {
            if (int(custom_exponents.size()) != r)
                throw DimensionError(detail::msg("SpectrumSpec: %zu custom exponents for rank %d",
                                                 custom_exponents.size(), r));
            exps = custom_exponents;
        } else {
            const double end = kind == Kind::kTypeI ? -0.5 : kind == Kind::kTypeII ? -2.0 : -3.5;
            exps.resize(std::size_t(r));
            if (r == 1)
                exps[0] = end;
            else
                for (int j = 0; j < r; ++j) exps[std::size_t(j)] = end * double(j) / (r - 1);
        }
        std::vector<double> sv(static_cast<std::size_t>(r));
        for (int j = 0; j < r; ++j) sv[std::size_t(j)] = std::pow(10.0, exps[std::size_t(j)]);
        return sv;
    }
};
struct TestMatrix {
    DenseMatrix a;
    std::vector<double> sigma_true;
};
// testmat.hpp:65-74 semantics on the GPU: U, V are orthonormalised Philox
// Gaussians keyed by one draw of `rng` (not the reference's RngState bits;
// the spectrum is exact).
inline TestMatrix gen_test_matrix(int m, int n, const SpectrumSpec& spec, RngState& rng) {
    TestMatrix out;
    out.sigma_true = spec.sigma(std::min(m, n));
    out.a = DenseMatrix(m, n);
    detail::check(rlra_gen_test_matrix(detail::ctx(), RLRA_HOST, m, n, out.sigma_true.data(),
                                       int(out.sigma_true.size()), rng.next_u64(), 0.0, out.a.data(),
                                       detail::ld(out.a)));
    return out;
}

// ------------------------------------------------------------ report.hpp ---
enum class FactorizationKind { kSvd, kId, kCur };
struct NnzCounts {
    std::vector<std::pair<std::string, double>> parts;
    double total = 0.0;
};
// report.hpp:30-58 storage accounting (plain arithmetic)
inline NnzCounts nnz_report(FactorizationKind kind, int m, int n, int k, double density = 1.0) {
    if (m < 1 || n < 1 || k < 1 || k > std::min(m, n))
        throw DimensionError(detail::msg("nnz_report: invalid shape m=%d n=%d k=%d", m, n, k));
    if (!(density > 0.0) || density > 1.0)
        throw DimensionError(detail::msg("nnz_report: density %g outside (0, 1]", density));
    const double dm = m, dn = n, dk = k;
    NnzCounts out;
    switch (kind) {
        case FactorizationKind::kSvd: out.parts = {{"U", dk * dm}, {"sigma", dk}, {"V", dk * dn}}; break;
        case FactorizationKind::kId:
            out.parts = {{"C", density * dk * dm}, {"V_interp", dk * (dn - dk)}, {"indices", dk}};
            break;
        case FactorizationKind::kCur:
            out.parts = {{"C", density * dk * dm}, {"U", dk * dk}, {"R", density * dk * dn}};
            break;
    }
    for (const auto& p : out.parts) out.total += p.second;
    return out;
}
struct ErrorReport {  // report.hpp:73-93
    std::string method;
    int m = 0, n = 0, k = 0;
    std::string params;
    double rel_frobenius_error = 0.0;
    double rel_spectral_error = 0.0;
    double fro_floor = std::numeric_limits<double>::quiet_NaN();
    double spec_floor = std::numeric_limits<double>::quiet_NaN();
    double spec_bound = std::numeric_limits<double>::quiet_NaN();
    NnzCounts nnz;
    double wall_seconds = 0.0;
};
namespace detail {
// verify_reconstruction (report.hpp:97-138) for recon = X Y^T on the GPU
inline ErrorReport verify_xyt(const DenseMatrix& a, const DenseMatrix& x, const DenseMatrix& y, int k,
                              const char* method, const std::vector<double>& sigma_true) {
    double out[5];
    check(rlra_verify_lowrank(ctx(), RLRA_HOST, a.data(), a.rows(), a.cols(), ld(a), x.data(), ld(x), y.data(), ld(y),
                              k, sigma_true.empty() ? nullptr : sigma_true.data(), int(sigma_true.size()), out));
    ErrorReport r;
    r.method = method;
    r.m = a.rows();
    r.n = a.cols();
    r.k = k;
    r.rel_frobenius_error = out[0];
    r.rel_spectral_error = out[1];
    r.fro_floor = out[2];
    r.spec_floor = out[3];
    r.spec_bound = out[4];
    return r;
}
}  // namespace detail
inline ErrorReport verify(const DenseMatrix& a, const SvdFactors& f, const std::vector<double>& sigma_true = {}) {
    if (f.u.rows() != a.rows() || f.v.rows() != a.cols() || f.u.cols() != f.k || f.v.cols() != f.k ||
        int(f.sigma.size()) != f.k)
        throw DimensionError("verify: SVD factor shapes do not match the matrix");
    DenseMatrix us = f.u;
    scale_columns_inplace(us, f.sigma);
    ErrorReport r = detail::verify_xyt(a, us, f.v, f.k, "svd", sigma_true);
    if (f.k > 0) r.nnz = nnz_report(FactorizationKind::kSvd, a.rows(), a.cols(), f.k);
    return r;
}
inline ErrorReport verify(const DenseMatrix& a, const IdFactors& f, const std::vector<double>& sigma_true = {}) {
    if (f.v.rows() != a.cols() || f.v.cols() != f.k || f.jc.size() != a.cols())
        throw DimensionError("verify: column-ID factor shapes do not match the matrix");
    ErrorReport r = detail::verify_xyt(a, select_columns(a, f.jc, f.k), f.v, f.k, "id", sigma_true);
    if (f.k > 0) r.nnz = nnz_report(FactorizationKind::kId, a.rows(), a.cols(), f.k);
    return r;
}
inline ErrorReport verify(const DenseMatrix& a, const RowIdFactors& f, const std::vector<double>& sigma_true = {}) {
    if (f.w.rows() != a.rows() || f.w.cols() != f.k || f.jr.size() != a.rows())
        throw DimensionError("verify: row-ID factor shapes do not match the matrix");
    ErrorReport r = detail::verify_xyt(a, f.w, transpose(select_rows(a, f.jr, f.k)), f.k, "id-row", sigma_true);
    if (f.k > 0) r.nnz = nnz_report(FactorizationKind::kId, a.cols(), a.rows(), f.k);
    return r;
}
inline ErrorReport verify(const DenseMatrix& a, const CurFactors& f, const std::vector<double>& sigma_true = {}) {
    if (f.c.rows() != a.rows() || f.r.cols() != a.cols() || f.c.cols() != f.k || f.r.rows() != f.k ||
        f.u.rows() != f.k || f.u.cols() != f.k)
        throw DimensionError("verify: CUR factor shapes do not match the matrix");
    ErrorReport r = detail::verify_xyt(a, f.c, transpose(matmul(f.u, f.r)), f.k, "cur", sigma_true);
    if (f.k > 0) r.nnz = nnz_report(FactorizationKind::kCur, a.rows(), a.cols(), f.k);
    return r;
}
inline ErrorReport verify(const DenseMatrix& a, const QbFactors& f, const std::vector<double>& sigma_true = {}) {
    if (f.q.rows() != a.rows() || f.b.cols() != a.cols() || f.q.cols() != f.ell || f.b.rows() != f.ell)
        throw DimensionError("verify: QB factor shapes do not match the matrix");
    ErrorReport r = detail::verify_xyt(a, f.q, transpose(f.b), f.ell, "qb", sigma_true);
    if (f.ell > 0) {
        const double dm = a.rows(), dn = a.cols(), dl = f.ell;
        r.nnz.parts = {{"Q", dl * dm}, {"B", dl * dn}};
        r.nnz.total = dl * (dm + dn);
    }
    return r;
}
// report.hpp:210-244 CSV emission
inline std::string csv_header() {
    return "method,m,n,k,params,rel_fro_error,rel_spec_error,fro_floor,spec_floor,spec_bound,nnz_total,seconds";
}
namespace detail {
inline std::string csv_num(double v) { return std::isnan(v) ? std::string() : msg("%.17g", v); }
}  // namespace detail
inline std::string csv_row(const ErrorReport& r) {
    std::string row = r.method;
    row += detail::msg(",%d,%d,%d,", r.m, r.n, r.k);
    row += r.params;
    for (double v : {r.rel_frobenius_error, r.rel_spectral_error, r.fro_floor, r.spec_floor, r.spec_bound,
                     r.nnz.total}) {
        row += ',';
        row += detail::csv_num(v);
    }
    row += detail::msg(",%.6f", r.wall_seconds);
    return row;
}

// ---------------------------------------------------- io.hpp: spectrum ---
inline void save_spectrum(const std::string& path, const std::vector<double>& sigma) {  // io.hpp:114-121
    FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw IoError(detail::msg("save_spectrum: cannot open '%s' for writing", path.c_str()));
    bool ok = true;
    for (double v : sigma) ok = ok && std::fprintf(f, "%.17g\n", v) > 0;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw IoError(detail::msg("save_spectrum: write to '%s' failed", path.c_str()));
}
inline std::vector<double> load_spectrum(const std::string& path) {  // io.hpp:123-147
    FILE* f = std::fopen(path.c_str(), "r");
    if (!f) throw IoError(detail::msg("load_spectrum: cannot open '%s'", path.c_str()));
    std::vector<double> sigma;
    std::string line;
    int lineno = 0, c = 0;
    bool more = true;
    while (more) {
        line.clear();
        while ((c = std::fgetc(f)) != EOF && c != '\n') line.push_back(char(c));
        more = c != EOF;
        if (!more && line.empty()) break;
        ++lineno;
        if (line.empty()) continue;
        const char* begin = line.c_str();
        char* end = nullptr;
        const double v = std::strtod(begin, &end);
        if (end == begin) {
            std::fclose(f);
            throw IoError(detail::msg("load_spectrum: '%s' line %d is not a number", path.c_str(), lineno));
        }
        std::size_t pos = std::size_t(end - begin);
        while (pos < line.size() && (line[pos] == ' ' || line[pos] == '\r')) ++pos;
        if (pos != line.size() || !std::isfinite(v)) {
            std::fclose(f);
            throw IoError(detail::msg("load_spectrum: '%s' line %d is not a finite number", path.c_str(), lineno));
        }
        sigma.push_back(v);
    }
    std::fclose(f);
    return sigma;
}

// ---------------------------------------------------- qb.hpp: qb_single ---
inline QbFactors qb_single(const DenseMatrix& a, double tol, int max_rank, RngState& rng) {  // qb.hpp:43-95
    const int m = a.rows(), n = a.cols();
    const int cap = std::max(1, max_rank);
    DenseMatrix Q(m, cap), B(cap, n);
    int ell = 0, reached = 0, nh = 0;
    double fin = 0.0;
    std::vector<double> hist(static_cast<std::size_t>(cap));
    rlra_omega om = detail::omega_from(rng, false);
    detail::check(rlra_qb_single(detail::ctx(), RLRA_HOST, a.data(), m, n, detail::ld(a), tol, max_rank, &om, Q.data(),
                                 std::max(1, m), B.data(), cap, &ell, hist.data(), &nh, &fin, &reached));
    QbFactors f;
    f.q = submatrix(Q, 0, m, 0, ell);
    f.b = submatrix(B, 0, ell, 0, n);
    f.ell = ell;
    f.residual_report.final_residual = fin;
    f.residual_report.tolerance_reached = reached != 0;
    f.residual_report.history.assign(hist.begin(), hist.begin() + nh);
    return f;
}

}  // namespace rlra
