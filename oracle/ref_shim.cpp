// ref_shim.cpp — C-ABI shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/rlra, compiled where they lie; nothing is
// copied).  TEST INFRASTRUCTURE: oracle/Makefile builds it into
// oracle/_ref/librlra_ref.so, which pins the C restatement (rlra_oracle.c)
// and serves as the "reference" CPU baseline in bench.py.  Signatures mirror
// rlra_oracle.h with a ref_ prefix; the rng is carried as the same plain
// struct so tests can hand identical states to both sides.
#include <cstring>
#include <string>

#include "rlra/rlra.hpp"

extern "C" {
struct ref_rng {
    std::uint64_t s[4];
    double spare;
    int have_spare;
};
}

namespace {
thread_local std::string g_err;

// RngState keeps its state private; the shim round-trips it through the
// seed-independent raw layout (4 x u64, double, bool), which is the class's
// only data.  A static_assert pins the size so a layout change fails to build.
static_assert(sizeof(rlra::RngState) == 48, "RngState layout changed");

rlra::RngState to_state(const ref_rng* r) {
    rlra::RngState s(0);
    unsigned char* p = reinterpret_cast<unsigned char*>(&s);
    std::memcpy(p, r->s, 32);
    std::memcpy(p + 32, &r->spare, 8);
    bool hs = r->have_spare != 0;
    std::memcpy(p + 40, &hs, 1);
    return s;
}

void from_state(const rlra::RngState& s, ref_rng* r) {
    const unsigned char* p = reinterpret_cast<const unsigned char*>(&s);
    std::memcpy(r->s, p, 32);
    std::memcpy(&r->spare, p + 32, 8);
    bool hs;
    std::memcpy(&hs, p + 40, 1);
    r->have_spare = hs ? 1 : 0;
}

rlra::DenseMatrix wrap(const double* a, int m, int n) {
    rlra::DenseMatrix x(m, n);
    if (m > 0 && n > 0) std::memcpy(x.data(), a, sizeof(double) * std::size_t(m) * n);
    return x;
}

void put(const rlra::DenseMatrix& x, double* out) {
    if (x.size()) std::memcpy(out, x.data(), sizeof(double) * x.size());
}

void put_cols(const rlra::DenseMatrix& x, double* out, int ld) {
    for (int j = 0; j < x.cols(); ++j)
        for (int i = 0; i < x.rows(); ++i) out[i + std::size_t(j) * ld] = x(i, j);
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const rlra::DimensionError& e) {
        g_err = e.what();
        return 1;
    } catch (const rlra::NumericalError& e) {
        g_err = e.what();
        return 2;
    } catch (const rlra::ConvergenceError& e) {
        g_err = e.what();
        return 3;
    } catch (const rlra::IoError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

void put_svd(const rlra::SvdFactors& f, double* u, double* sigma, double* v) {
    put(f.u, u);
    put(f.v, v);
    std::memcpy(sigma, f.sigma.data(), sizeof(double) * f.sigma.size());
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { rlra::config::set_threads(n); }

void ref_rng_seed(ref_rng* r, std::uint64_t seed) { from_state(rlra::RngState(seed), r); }

void ref_gaussian_matrix(int rows, int cols, ref_rng* r, double* out) {
    rlra::RngState s = to_state(r);
    put(rlra::gaussian_matrix(rows, cols, s), out);
    from_state(s, r);
}

void ref_rng_substream(ref_rng* parent, ref_rng* child) {
    rlra::RngState s = to_state(parent);
    rlra::RngState c = s.substream();
    from_state(s, parent);
    from_state(c, child);
}

int ref_matmul(int ta, int tb, const double* a, int ar, int ac, const double* b, int br, int bc,
               double* c) {
    return guard([&] { put(rlra::matmul(wrap(a, ar, ac), wrap(b, br, bc), ta, tb), c); });
}

int ref_compact_qr(const double* a, int m, int n, double* q, double* r, int* degenerate) {
    return guard([&] {
        rlra::QrFactors f = rlra::compact_qr(wrap(a, m, n));
        put(f.q, q);
        put(f.r, r);
        if (degenerate) *degenerate = f.degenerate_rank;
    });
}

int ref_pivoted_qr(const double* a, int m, int n, int k, double tol, double* q1, double* s1,
                   int ld_s1, int* perm, int* frank, double* residual, int* reached,
                   int* degenerate) {
    return guard([&] {
        rlra::PivotedQr f = rlra::pivoted_qr_partial(wrap(a, m, n), k, tol);
        put(f.q1, q1);
        put_cols(f.s1, s1, ld_s1);
        for (int j = 0; j < n; ++j) perm[j] = f.perm[j];
        *frank = f.frank;
        *residual = f.residual;
        *reached = f.tolerance_reached;
        if (degenerate) *degenerate = f.degenerate_rank;
    });
}

int ref_upper_tri_solve(const double* s11, int k, const double* s12, int nc, double* t,
                        int* clamped) {
    return guard([&] {
        rlra::TriSolve ts = rlra::upper_tri_solve(wrap(s11, k, k), wrap(s12, k, nc));
        put(ts.t, t);
        *clamped = ts.clamped;
    });
}

int ref_small_svd(const double* a, int m, int n, double* u, double* sigma, double* v) {
    return guard([&] { put_svd(rlra::small_svd(wrap(a, m, n)), u, sigma, v); });
}

int ref_sym_eig(const double* t, int n, double* values, double* vectors) {
    return guard([&] {
        rlra::SymEig e = rlra::sym_eig(wrap(t, n, n));
        std::memcpy(values, e.values.data(), sizeof(double) * n);
        put(e.vectors, vectors);
    });
}

int ref_sample(int left, const double* a, int m, int n, int l, int q, int s, ref_rng* r,
               double* y) {
    return guard([&] {
        rlra::RngState st = to_state(r);
        rlra::DenseMatrix A = wrap(a, m, n);
        put(left ? rlra::sample_left(A, l, q, s, st) : rlra::sample_right(A, l, q, s, st), y);
        from_state(st, r);
    });
}

int ref_rsvd(int variant, const double* a, int m, int n, int k, int p, int q, int s, ref_rng* r,
             double* u, double* sigma, double* v) {
    return guard([&] {
        rlra::RngState st = to_state(r);
        rlra::DenseMatrix A = wrap(a, m, n);
        rlra::SvdFactors f = variant == 0   ? rlra::rsvd_v2(A, k, p, q, s, st)
                             : variant == 1 ? rlra::rsvd_v1(A, k, p, q, s, st)
                                            : rlra::rsvd_basic(A, k, p, st);
        put_svd(f, u, sigma, v);
        from_state(st, r);
    });
}

int ref_qb_blocked(const double* a, int m, int n, int blk, int num_blocks, double tol, int q_power,
                   int reorth, ref_rng* r, double* Q, double* B, int cap, int* ell, double* hist,
                   int* nhist, double* final_resid, int* reached, double* w_out) {
    return guard([&] {
        rlra::RngState st = to_state(r);
        rlra::DenseMatrix W = wrap(a, m, n);
        rlra::QbFactors f = rlra::qb_blocked_inplace(W, blk, num_blocks, tol, q_power, reorth, st);
        put(f.q, Q);
        put_cols(f.b, B, cap);
        *ell = f.ell;
        *nhist = int(f.residual_report.history.size());
        for (int i = 0; i < *nhist; ++i) hist[i] = f.residual_report.history[i];
        *final_resid = f.residual_report.final_residual;
        *reached = f.residual_report.tolerance_reached;
        if (w_out) put(W, w_out);
        from_state(st, r);
    });
}

int ref_svd_from_qb(const double* q, const double* b, int ldb, int m, int n, int ell, int k,
                    int vnum, double* u, double* sigma, double* v, int* k_out) {
    return guard([&] {
        rlra::QbFactors f;
        f.q = wrap(q, m, ell);
        f.b = rlra::DenseMatrix(ell, n);
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < ell; ++i) f.b(i, j) = b[i + std::size_t(j) * ldb];
        f.ell = ell;
        rlra::SvdFactors s = rlra::svd_from_qb(f, k, vnum ? rlra::Vnum::kBbt : rlra::Vnum::kQr);
        put_svd(s, u, sigma, v);
        *k_out = s.k;
    });
}

int ref_id_column(const double* a, int m, int n, int k, double tol, int* jc, double* v, int* k_out,
                  double* qr_residual, int* reached, int* clamped) {
    return guard([&] {
        rlra::IdFactors f = rlra::id_column(wrap(a, m, n), k, tol);
        for (int j = 0; j < n; ++j) jc[j] = f.jc[j];
        put(f.v, v);
        *k_out = f.k;
        *qr_residual = f.qr_residual;
        *reached = f.tolerance_reached;
        *clamped = f.clamped;
    });
}

int ref_id_rand(const double* a, int m, int n, int k, int p, int q, int s, ref_rng* r, int* jc,
                double* v, double* qr_residual, int* clamped) {
    return guard([&] {
        rlra::RngState st = to_state(r);
        rlra::IdFactors f = rlra::id_rand(wrap(a, m, n), k, p, q, s, st);
        for (int j = 0; j < n; ++j) jc[j] = f.jc[j];
        put(f.v, v);
        *qr_residual = f.qr_residual;
        *clamped = f.clamped;
        from_state(st, r);
    });
}

int ref_cur_rand(const double* a, int m, int n, int k, int p, int q, int s, ref_rng* r, int* jc,
                 int* jr, double* c, double* u, double* rr, double* residual,
                 double* qr_residual) {
    return guard([&] {
        rlra::RngState st = to_state(r);
        rlra::CurFactors f = rlra::cur_rand(wrap(a, m, n), k, p, q, s, st);
        for (int j = 0; j < n; ++j) jc[j] = f.jc[j];
        for (int i = 0; i < m; ++i) jr[i] = f.jr[i];
        put(f.c, c);
        put(f.u, u);
        put(f.r, rr);
        *residual = f.residual;
        *qr_residual = f.qr_residual;
        from_state(st, r);
    });
}

int ref_two_sided_from_column(const double* a, int m, int n, const int* jc, const double* v, int k,
                              int* jr, double* w) {
    return guard([&] {
        rlra::IdFactors col;
        col.jc = rlra::Permutation(std::vector<int>(jc, jc + n));
        col.v = wrap(v, n, k);
        col.k = k;
        rlra::TwoSidedIdFactors t = rlra::detail::two_sided_from_column(wrap(a, m, n), col);
        for (int i = 0; i < m; ++i) jr[i] = t.jr[i];
        put(t.w, w);
    });
}

// qb.hpp qb_parallel / qb_hierarchical: q m x ell, b ell x n (ld ell)
int ref_qb_parallel(const double* a, int m, int n, int blk, int num_blocks, int q_power, ref_rng* r, double* q,
                    double* b, double* final_resid) {
    return guard([&] {
        rlra::RngState st = to_state(r);
        rlra::QbFactors f = rlra::qb_parallel(wrap(a, m, n), blk, num_blocks, q_power, st);
        put(f.q, q);
        put(f.b, b);
        *final_resid = f.residual_report.final_residual;
        from_state(st, r);
    });
}

int ref_qb_hierarchical(const double* a, int m, int n, int nrb, int blk, int num_blocks, int q_power, ref_rng* r,
                        double* q, double* b, double* final_resid) {
    return guard([&] {
        rlra::RngState st = to_state(r);
        rlra::QbFactors f = rlra::qb_hierarchical(wrap(a, m, n), nrb, blk, num_blocks, q_power, st);
        put(f.q, q);
        put(f.b, b);
        *final_resid = f.residual_report.final_residual;
        from_state(st, r);
    });
}

// report.hpp verify(a, SvdFactors, sigma_true): out = rel_fro, rel_spec,
// fro_floor, spec_floor, spec_bound
int ref_verify_svd(const double* a, int m, int n, const double* u, const double* sigma, const double* v, int k,
                   const double* sigma_true, int r, double* out) {
    return guard([&] {
        rlra::SvdFactors f;
        f.u = wrap(u, m, k);
        f.v = wrap(v, n, k);
        f.sigma.assign(sigma, sigma + k);
        f.k = k;
        std::vector<double> st;
        if (r > 0) st.assign(sigma_true, sigma_true + r);
        rlra::ErrorReport rep = rlra::verify(wrap(a, m, n), f, st);
        out[0] = rep.rel_frobenius_error;
        out[1] = rep.rel_spectral_error;
        out[2] = rep.fro_floor;
        out[3] = rep.spec_floor;
        out[4] = rep.spec_bound;
    });
}

// io.hpp save_binary / load_binary (row-major file <-> column-major buffer)
int ref_save_binary(const char* path, const double* a, int m, int n) {
    return guard([&] { rlra::save_binary(path, wrap(a, m, n)); });
}

int ref_load_binary(const char* path, int* rows, int* cols, double* out) {
    return guard([&] {
        rlra::DenseMatrix A = rlra::load_binary(path);
        *rows = A.rows();
        *cols = A.cols();
        if (out) put(A, out);
    });
}

}  // extern "C"
