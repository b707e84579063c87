/*
 * rlra_oracle.c — CPU restatement of the reference's randomized low-rank
 * factorization path.  TEST INFRASTRUCTURE: the parity checker, never the
 * product (see rlra_oracle.h).  Each function names the reference lines it
 * restates; paths are relative to /root/reference/proj/include/rlra/.
 *
 * Bit-identity with the reference needs the same flags on both sides
 * (oracle/Makefile: -O2 -ffp-contract=off), the same libm, and the same
 * evaluation order, which is why the loops below keep the reference's
 * order even where a faster order exists.
 */
#include "rlra_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EDIM 1
#define ORC_ENUM 2
#define ORC_ECONV 3

static _Thread_local char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

#define IDX(i, j, ld) ((size_t)(i) + (size_t)(j) * (size_t)(ld))

static double* dalloc(size_t n) {
    double* p = (double*)calloc(n ? n : 1, sizeof(double));
    if (!p) abort();
    return p;
}

/* ------------------------------------------------------------------ rng --- */
/* core/rng.hpp:66-74 splitmix64 */
static uint64_t splitmix64(uint64_t* x) {
    uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* core/rng.hpp:20-24 */
void orc_rng_seed(orc_rng* r, uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&x);
    r->spare = 0.0;
    r->have_spare = 0;
}

/* core/rng.hpp:27-38 xoshiro256++ */
uint64_t orc_rng_next_u64(orc_rng* r) {
    uint64_t* s = r->s;
    const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

static double next_unit(orc_rng* r) { return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53; }

/* core/rng.hpp:43-56 Box-Muller with a cached spare */
double orc_rng_gaussian(orc_rng* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    const double u1 = 1.0 - next_unit(r);
    const double u2 = next_unit(r);
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * 3.14159265358979323846 * u2;
    r->spare = radius * sin(angle);
    r->have_spare = 1;
    return radius * cos(angle);
}

/* core/rng.hpp:61-64 */
void orc_rng_substream(orc_rng* parent, orc_rng* child) {
    uint64_t key = orc_rng_next_u64(parent);
    orc_rng_seed(child, splitmix64(&key));
}

/* core/rng.hpp:82-87: column-major fill */
void orc_gaussian_matrix(int rows, int cols, orc_rng* r, double* out) {
    const size_t n = (size_t)rows * (size_t)cols;
    for (size_t i = 0; i < n; ++i) out[i] = orc_rng_gaussian(r);
}

/* --------------------------------------------------------------- matmul --- */
/* core/matmul.hpp:16-61.  Column j of c only depends on column j's loop, so
 * this single-threaded restatement equals the threaded reference bitwise. */
static void mm(int ta, int tb, const double* a, int ar, int ac, const double* b, int br, int bc,
               double* c, int m, int n) {
    const int inner = ta ? ar : ac;
    (void)ac;
    (void)bc;
    memset(c, 0, sizeof(double) * (size_t)m * (size_t)n);
    if (!ta && !tb) {
        for (int j = 0; j < n; ++j) {
            double* cj = c + IDX(0, j, m);
            const double* bj = b + IDX(0, j, br);
            for (int l = 0; l < inner; ++l) {
                const double blj = bj[l];
                const double* al = a + IDX(0, l, ar);
                for (int i = 0; i < m; ++i) cj[i] += al[i] * blj;
            }
        }
    } else if (ta && !tb) {
        for (int j = 0; j < n; ++j) {
            double* cj = c + IDX(0, j, m);
            const double* bj = b + IDX(0, j, br);
            for (int i = 0; i < m; ++i) {
                const double* ai = a + IDX(0, i, ar);
                double sum = 0.0;
                for (int l = 0; l < inner; ++l) sum += ai[l] * bj[l];
                cj[i] = sum;
            }
        }
    } else if (!ta && tb) {
        for (int j = 0; j < n; ++j) {
            double* cj = c + IDX(0, j, m);
            for (int l = 0; l < inner; ++l) {
                const double bjl = b[IDX(j, l, br)];
                const double* al = a + IDX(0, l, ar);
                for (int i = 0; i < m; ++i) cj[i] += al[i] * bjl;
            }
        }
    } else {
        for (int j = 0; j < n; ++j) {
            double* cj = c + IDX(0, j, m);
            for (int i = 0; i < m; ++i) {
                const double* ai = a + IDX(0, i, ar);
                double sum = 0.0;
                for (int l = 0; l < inner; ++l) sum += ai[l] * b[IDX(j, l, br)];
                cj[i] = sum;
            }
        }
    }
}

/* core/matmul.hpp:68-95 */
int orc_matmul(int ta, int tb, const double* a, int ar, int ac, const double* b, int br, int bc,
               double* c) {
    const int m = ta ? ac : ar;
    const int ka = ta ? ar : ac;
    const int kb = tb ? bc : br;
    const int n = tb ? br : bc;
    if (ka != kb)
        return fail(ORC_EDIM, "matmul: inner dimensions disagree: op(%dx%d) * op(%dx%d)", ar, ac,
                    br, bc);
    mm(ta, tb, a, ar, ac, b, br, bc, c, m, n);
    return ORC_OK;
}

/* ---------------------------------------------------------------- norms --- */
/* core/norms.hpp:14-25 Kahan-compensated sum of squares */
double orc_sum_squares(const double* p, int64_t n) {
    double sum = 0.0, comp = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double term = p[i] * p[i];
        const double y = term - comp;
        const double t = sum + y;
        comp = (t - sum) - y;
        sum = t;
    }
    return sum;
}

double orc_frobenius(const double* a, int64_t count) { return sqrt(orc_sum_squares(a, count)); }

/* ------------------------------------------------------------ householder --- */
/* core/qr.hpp:44-66.  w is m x ?, ld m; v_store m x ?, ld m. */
static double householder_step(double* w, int m, int row0, int col, double* v_store) {
    double norm2 = 0.0;
    double* wc = w + IDX(0, col, m);
    double* vc = v_store + IDX(0, col, m);
    for (int i = row0; i < m; ++i) norm2 += wc[i] * wc[i];
    const double norm = sqrt(norm2);
    for (int i = 0; i < m; ++i) vc[i] = 0.0;
    if (norm < 1e-300) {
        wc[row0] = 0.0;
        for (int i = row0 + 1; i < m; ++i) wc[i] = 0.0;
        return 0.0;
    }
    const double x1 = wc[row0];
    const double alpha = x1 >= 0.0 ? -norm : norm;
    for (int i = row0; i < m; ++i) vc[i] = wc[i];
    vc[row0] -= alpha;
    const double vnorm2 = 2.0 * (norm2 - alpha * x1);
    wc[row0] = alpha;
    for (int i = row0 + 1; i < m; ++i) wc[i] = 0.0;
    return 2.0 / vnorm2;
}

/* core/qr.hpp:69-79 */
static void apply_reflector(double* w, int m, const double* v_store, double beta, int row0,
                            int refl_col, int j) {
    if (beta == 0.0) return;
    const double* v = v_store + IDX(0, refl_col, m);
    double* wj = w + IDX(0, j, m);
    double dot = 0.0;
    for (int i = row0; i < m; ++i) dot += v[i] * wj[i];
    const double f = beta * dot;
    for (int i = row0; i < m; ++i) wj[i] -= f * v[i];
}

/* core/qr.hpp:82-89 */
static void form_q(const double* v_store, const double* betas, int nb, int m, int cols, double* q) {
    memset(q, 0, sizeof(double) * (size_t)m * (size_t)cols);
    for (int j = 0; j < cols; ++j) q[IDX(j, j, m)] = 1.0;
    for (int k = nb - 1; k >= 0; --k)
        for (int j = 0; j < cols; ++j) apply_reflector(q, m, v_store, betas[k], k, k, j);
}

/* core/qr.hpp:95-121 */
int orc_compact_qr(const double* a, int m, int n, double* q, double* r, int* degenerate) {
    if (m < n) return fail(ORC_EDIM, "compact_qr: matrix is %dx%d, need rows >= cols", m, n);
    double* w = dalloc((size_t)m * n);
    double* vs = dalloc((size_t)m * n);
    double* betas = dalloc((size_t)n);
    memcpy(w, a, sizeof(double) * (size_t)m * n);
    int deg = 0;
    for (int k = 0; k < n; ++k) {
        betas[k] = householder_step(w, m, k, k, vs);
        if (betas[k] == 0.0) deg = 1;
        for (int j = k + 1; j < n; ++j) apply_reflector(w, m, vs, betas[k], k, k, j);
    }
    form_q(vs, betas, n, m, n, q);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) r[IDX(i, j, n)] = w[IDX(i, j, m)];
    for (int k = 0; k < n; ++k) {
        if (r[IDX(k, k, n)] < 0.0) {
            for (int j = k; j < n; ++j) r[IDX(k, j, n)] = -r[IDX(k, j, n)];
            for (int i = 0; i < m; ++i) q[IDX(i, k, m)] = -q[IDX(i, k, m)];
        }
    }
    if (degenerate) *degenerate = deg;
    free(w);
    free(vs);
    free(betas);
    return ORC_OK;
}

static int orth_inplace(double* y, int m, int n) {
    double* q = dalloc((size_t)m * n);
    double* r = dalloc((size_t)n * n);
    int st = orc_compact_qr(y, m, n, q, r, NULL);
    if (st == ORC_OK) memcpy(y, q, sizeof(double) * (size_t)m * n);
    free(q);
    free(r);
    return st;
}

/* ----------------------------------------------------------- pivoted QR --- */
/* core/qr.hpp:140-236 */
int orc_pivoted_qr(const double* a, int m, int n, int k, double tol, double* q1, double* s1,
                   int ld_s1, int* perm, int* frank_out, double* residual_out, int* reached_out,
                   int* degenerate_out) {
    const int rmax = m < n ? m : n;
    const int tol_mode = (k == 0 && tol > 0.0);
    if (!tol_mode && (k < 1 || k > rmax || tol != 0.0))
        return fail(ORC_EDIM,
                    "pivoted_qr_partial: need either k in [1,%d] with tol=0 or k=0 with tol>0 "
                    "(got k=%d, tol=%g)",
                    rmax, k, tol);
    const int kmax = tol_mode ? rmax : k;
    double* w = dalloc((size_t)m * n);
    double* vs = dalloc((size_t)m * (kmax > 0 ? kmax : 1));
    double* betas = dalloc((size_t)kmax + 1);
    double* cn = dalloc((size_t)n);
    double* rn = dalloc((size_t)n);
    memcpy(w, a, sizeof(double) * (size_t)m * n);
    for (int j = 0; j < n; ++j) {
        perm[j] = j;
        cn[j] = orc_sum_squares(w + IDX(0, j, m), m);
        rn[j] = cn[j];
    }
#define TRAILING_NORM(f, out)                                                   \
    do {                                                                        \
        double s_ = 0.0;                                                        \
        for (int jj = (f); jj < n; ++jj) s_ += orc_sum_squares(w + IDX((f), jj, m), m - (f)); \
        (out) = sqrt(s_);                                                       \
    } while (0)
    int deg = 0, frank = 0;
    double residual = 0.0;
    if (tol_mode) TRAILING_NORM(0, residual);
    int reached = tol_mode && residual <= tol;
    while (!reached && frank < kmax) {
        const int f = frank;
        int piv = f;
        for (int j = f + 1; j < n; ++j)
            if (cn[j] > cn[piv]) piv = j;
        if (piv != f) {
            for (int i = 0; i < m; ++i) {
                double t = w[IDX(i, f, m)];
                w[IDX(i, f, m)] = w[IDX(i, piv, m)];
                w[IDX(i, piv, m)] = t;
            }
            int ti = perm[f]; perm[f] = perm[piv]; perm[piv] = ti;
            double td = cn[f]; cn[f] = cn[piv]; cn[piv] = td;
            td = rn[f]; rn[f] = rn[piv]; rn[piv] = td;
        }
        /* v_store is m x kmax; reflector f lives in its column f. */
        betas[f] = 0.0;
        {
            /* householder_step writes v_store(:, col=f) and w(:, f) */
            double norm2 = 0.0;
            double* wc = w + IDX(0, f, m);
            double* vc = vs + IDX(0, f, m);
            for (int i = f; i < m; ++i) norm2 += wc[i] * wc[i];
            const double norm = sqrt(norm2);
            for (int i = 0; i < m; ++i) vc[i] = 0.0;
            if (norm < 1e-300) {
                wc[f] = 0.0;
                for (int i = f + 1; i < m; ++i) wc[i] = 0.0;
                betas[f] = 0.0;
            } else {
                const double x1 = wc[f];
                const double alpha = x1 >= 0.0 ? -norm : norm;
                for (int i = f; i < m; ++i) vc[i] = wc[i];
                vc[f] -= alpha;
                const double vnorm2 = 2.0 * (norm2 - alpha * x1);
                wc[f] = alpha;
                for (int i = f + 1; i < m; ++i) wc[i] = 0.0;
                betas[f] = 2.0 / vnorm2;
            }
        }
        if (betas[f] == 0.0) deg = 1;
        for (int j = f + 1; j < n; ++j) apply_reflector(w, m, vs, betas[f], f, f, j);
        for (int j = f + 1; j < n; ++j) {
            const double d = w[IDX(f, j, m)];
            cn[j] -= d * d;
            if (cn[j] < 1e-6 * rn[j]) {
                cn[j] = orc_sum_squares(w + IDX(f + 1, j, m), m - f - 1);
                rn[j] = cn[j];
            }
        }
        ++frank;
        if (tol_mode && frank < rmax) {
            TRAILING_NORM(frank, residual);
            if (residual <= tol) reached = 1;
        }
    }
    /* q1 = form_q(v_store, betas, m, frank); s1 = w(0:frank, :) */
    form_q(vs, betas, frank, m, frank, q1);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < frank; ++i) s1[IDX(i, j, ld_s1)] = w[IDX(i, j, m)];
    for (int kk = 0; kk < frank; ++kk) {
        if (s1[IDX(kk, kk, ld_s1)] < 0.0) {
            for (int j = kk; j < n; ++j) s1[IDX(kk, j, ld_s1)] = -s1[IDX(kk, j, ld_s1)];
            for (int i = 0; i < m; ++i) q1[IDX(i, kk, m)] = -q1[IDX(i, kk, m)];
        }
    }
    if (!tol_mode) {
        TRAILING_NORM(frank, residual);
        *reached_out = 0;
    } else if (reached) {
        *reached_out = 1;
    } else {
        /* ||A(:,perm) - Q1 S1||_F */
        double* diff = dalloc((size_t)m * n);
        double* s1c = dalloc((size_t)frank * n + 1);
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < frank; ++i) s1c[IDX(i, j, frank)] = s1[IDX(i, j, ld_s1)];
        mm(0, 0, q1, m, frank, s1c, frank, n, diff, m, n);
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < m; ++i)
                diff[IDX(i, j, m)] = a[IDX(i, perm[j], m)] - diff[IDX(i, j, m)];
        residual = orc_frobenius(diff, (int64_t)m * n);
        *reached_out = residual <= tol;
        free(diff);
        free(s1c);
    }
#undef TRAILING_NORM
    *frank_out = frank;
    *residual_out = residual;
    if (degenerate_out) *degenerate_out = deg;
    free(w);
    free(vs);
    free(betas);
    free(cn);
    free(rn);
    return ORC_OK;
}

/* --------------------------------------------------------- tri-solve --- */
/* core/qr.hpp:242-275 */
int orc_upper_tri_solve(const double* s11, int lds11, int k, const double* s12, int lds12, int nc,
                        double* t, int* clamped) {
    double dmax = 0.0, dmin = INFINITY;
    for (int i = 0; i < k; ++i) {
        const double d = fabs(s11[IDX(i, i, lds11)]);
        if (d == 0.0) return fail(ORC_ENUM, "upper_tri_solve: zero diagonal at position %d", i);
        if (d > dmax) dmax = d;
        if (d < dmin) dmin = d;
    }
    for (int j = 0; j < nc; ++j) {
        double* tj = t + IDX(0, j, k);
        const double* bj = s12 + IDX(0, j, lds12);
        for (int i = k - 1; i >= 0; --i) {
            double sum = bj[i];
            for (int l = i + 1; l < k; ++l) sum -= s11[IDX(i, l, lds11)] * tj[l];
            tj[i] = sum / s11[IDX(i, i, lds11)];
        }
    }
    *clamped = 0;
    if (k > 0 && dmax / dmin > 1e12) {
        *clamped = 1;
        const size_t cnt = (size_t)k * nc;
        for (size_t i = 0; i < cnt; ++i)
            if (fabs(t[i]) > 1e4) t[i] = t[i] > 0.0 ? 1e4 : -1e4;
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------- jacobi --- */
/* core/jacobi.hpp:33-60 */
static void complete_column(double* u, int m, const int* done, int ndone, int j) {
    int best = 0;
    double best_resid = -1.0;
    for (int i = 0; i < m; ++i) {
        double proj2 = 0.0;
        for (int c = 0; c < ndone; ++c) proj2 += u[IDX(i, done[c], m)] * u[IDX(i, done[c], m)];
        const double resid = 1.0 - proj2;
        if (resid > best_resid) {
            best_resid = resid;
            best = i;
        }
    }
    double* r = dalloc((size_t)m);
    r[best] = 1.0;
    for (int pass = 0; pass < 2; ++pass) {
        for (int c = 0; c < ndone; ++c) {
            const double* uc = u + IDX(0, done[c], m);
            double dot = 0.0;
            for (int i = 0; i < m; ++i) dot += uc[i] * r[i];
            for (int i = 0; i < m; ++i) r[i] -= dot * uc[i];
        }
    }
    double norm = 0.0;
    for (int i = 0; i < m; ++i) norm += r[i] * r[i];
    norm = sqrt(norm);
    for (int i = 0; i < m; ++i) u[IDX(i, j, m)] = r[i] / norm;
    free(r);
}

/* stable descending order of keys (std::stable_sort with '>' comparator) */
static void stable_order_desc(const double* key, int n, int* order) {
    for (int i = 0; i < n; ++i) order[i] = i;
    /* insertion sort is stable; n is small (<= a few thousand) */
    for (int i = 1; i < n; ++i) {
        int x = order[i];
        int j = i - 1;
        while (j >= 0 && key[x] > key[order[j]]) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = x;
    }
}

/* core/jacobi.hpp:145-232 (m >= n branch); u m x n, v n x n */
static int small_svd_tall(const double* a, int m, int n, double* u, double* sigma, double* v) {
    double* w = dalloc((size_t)m * n);
    double* vv = dalloc((size_t)n * n);
    memcpy(w, a, sizeof(double) * (size_t)m * n);
    for (int i = 0; i < n; ++i) vv[IDX(i, i, n)] = 1.0;
    const double eps = 1e-15;
    int sweep = 0;
    int rotated = n > 1;
    while (rotated) {
        if (sweep++ >= 60) {
            free(w);
            free(vv);
            return fail(ORC_ECONV, "small_svd: no convergence after %d sweeps on %dx%d input", 60,
                        m, n);
        }
        rotated = 0;
        for (int p = 0; p < n - 1; ++p) {
            for (int q = p + 1; q < n; ++q) {
                double app = 0.0, aqq = 0.0, apq = 0.0;
                double* wp = w + IDX(0, p, m);
                double* wq = w + IDX(0, q, m);
                for (int i = 0; i < m; ++i) {
                    app += wp[i] * wp[i];
                    aqq += wq[i] * wq[i];
                    apq += wp[i] * wq[i];
                }
                if (app == 0.0 || aqq == 0.0) continue;
                if (fabs(apq) <= eps * sqrt(app * aqq)) continue;
                const double zeta = (aqq - app) / (2.0 * apq);
                const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + tt * tt);
                const double s = tt * c;
                for (int i = 0; i < m; ++i) {
                    const double xp = wp[i];
                    const double xq = wq[i];
                    wp[i] = c * xp - s * xq;
                    wq[i] = s * xp + c * xq;
                }
                double* vp = vv + IDX(0, p, n);
                double* vq = vv + IDX(0, q, n);
                for (int i = 0; i < n; ++i) {
                    const double xp = vp[i];
                    const double xq = vq[i];
                    vp[i] = c * xp - s * xq;
                    vq[i] = s * xp + c * xq;
                }
                rotated = 1;
            }
        }
    }
    double* sg = dalloc((size_t)n);
    int* order = (int*)malloc(sizeof(int) * (size_t)(n ? n : 1));
    int* filled = (int*)malloc(sizeof(int) * (size_t)(n ? n : 1));
    int* needs = (int*)malloc(sizeof(int) * (size_t)(n ? n : 1));
    for (int j = 0; j < n; ++j) sg[j] = sqrt(orc_sum_squares(w + IDX(0, j, m), m));
    stable_order_desc(sg, n, order);
    memset(u, 0, sizeof(double) * (size_t)m * n);
    int nf = 0, nn = 0;
    for (int j = 0; j < n; ++j) {
        const int src = order[j];
        sigma[j] = sg[src];
        for (int i = 0; i < n; ++i) v[IDX(i, j, n)] = vv[IDX(i, src, n)];
        if (sg[src] > 1e-300) {
            for (int i = 0; i < m; ++i) u[IDX(i, j, m)] = w[IDX(i, src, m)] / sg[src];
            filled[nf++] = j;
        } else {
            sigma[j] = 0.0;
            needs[nn++] = j;
        }
    }
    for (int t = 0; t < nn; ++t) {
        complete_column(u, m, filled, nf, needs[t]);
        filled[nf++] = needs[t];
    }
    free(w);
    free(vv);
    free(sg);
    free(order);
    free(filled);
    free(needs);
    return ORC_OK;
}

/* core/jacobi.hpp:145-152: wide inputs go through the transpose */
int orc_small_svd(const double* a, int m, int n, double* u, double* sigma, double* v) {
    if (m >= n) return small_svd_tall(a, m, n, u, sigma, v);
    double* at = dalloc((size_t)m * n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < m; ++i) at[IDX(j, i, n)] = a[IDX(i, j, m)];
    /* small_svd(A^T): u' n x m, v' m x m; swap roles */
    int st = small_svd_tall(at, n, m, v, sigma, u);
    free(at);
    return st;
}

/* core/jacobi.hpp:68-139 */
int orc_sym_eig(const double* t, int n, double* values, double* vectors) {
    const double tnorm = orc_frobenius(t, (int64_t)n * n);
    double asym = 0.0;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < j; ++i) {
            double d = fabs(t[IDX(i, j, n)] - t[IDX(j, i, n)]);
            if (d > asym) asym = d;
        }
    if (tnorm > 0.0 && asym > 1e-12 * tnorm)
        return fail(ORC_ENUM, "sym_eig: asymmetry %.3e exceeds 1e-12 relative to norm %.3e", asym,
                    tnorm);
    double* mx = dalloc((size_t)n * n);
    double* u = dalloc((size_t)n * n);
    memcpy(mx, t, sizeof(double) * (size_t)n * n);
    for (int i = 0; i < n; ++i) u[IDX(i, i, n)] = 1.0;
#define OFFDIAG(out)                                                            \
    do {                                                                        \
        double s_ = 0.0;                                                        \
        for (int jj = 0; jj < n; ++jj)                                          \
            for (int ii = 0; ii < jj; ++ii) s_ += 2.0 * mx[IDX(ii, jj, n)] * mx[IDX(ii, jj, n)]; \
        (out) = sqrt(s_);                                                       \
    } while (0)
    int sweep = 0;
    double off;
    const double thr = 1e-14 * (tnorm > 1e-300 ? tnorm : 1e-300);
    for (;;) {
        if (n <= 1) break;
        OFFDIAG(off);
        if (!(off > thr)) break;
        if (sweep++ >= 30) {
            free(mx);
            free(u);
            return fail(ORC_ECONV,
                        "sym_eig: no convergence after %d sweeps; off-diagonal norm %.3e (matrix "
                        "norm %.3e)",
                        30, off, tnorm);
        }
        for (int p = 0; p < n - 1; ++p) {
            for (int q = p + 1; q < n; ++q) {
                const double apq = mx[IDX(p, q, n)];
                if (fabs(apq) <= 1e-300) continue;
                const double theta = (mx[IDX(q, q, n)] - mx[IDX(p, p, n)]) / (2.0 * apq);
                const double tt = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
                const double c = 1.0 / sqrt(1.0 + tt * tt);
                const double s = tt * c;
                for (int i = 0; i < n; ++i) {
                    const double mip = mx[IDX(i, p, n)];
                    const double miq = mx[IDX(i, q, n)];
                    mx[IDX(i, p, n)] = c * mip - s * miq;
                    mx[IDX(i, q, n)] = s * mip + c * miq;
                }
                for (int i = 0; i < n; ++i) {
                    const double mpi = mx[IDX(p, i, n)];
                    const double mqi = mx[IDX(q, i, n)];
                    mx[IDX(p, i, n)] = c * mpi - s * mqi;
                    mx[IDX(q, i, n)] = s * mpi + c * mqi;
                }
                for (int i = 0; i < n; ++i) {
                    const double uip = u[IDX(i, p, n)];
                    const double uiq = u[IDX(i, q, n)];
                    u[IDX(i, p, n)] = c * uip - s * uiq;
                    u[IDX(i, q, n)] = s * uip + c * uiq;
                }
            }
        }
    }
#undef OFFDIAG
    double* diag = dalloc((size_t)n);
    int* order = (int*)malloc(sizeof(int) * (size_t)(n ? n : 1));
    for (int i = 0; i < n; ++i) diag[i] = mx[IDX(i, i, n)];
    stable_order_desc(diag, n, order);
    for (int j = 0; j < n; ++j) {
        values[j] = diag[order[j]];
        for (int i = 0; i < n; ++i) vectors[IDX(i, j, n)] = u[IDX(i, order[j], n)];
    }
    free(mx);
    free(u);
    free(diag);
    free(order);
    return ORC_OK;
}

/* ---------------------------------------------------------------- sketch --- */
/* sketch.hpp:44-60 */
int orc_sample_right(const double* a, int m, int n, int l, int q, int s, orc_rng* r, double* y) {
    const int min_dim = m < n ? m : n;
    if (l < 1 || l > min_dim)
        return fail(ORC_EDIM, "sample_right: width %d out of range [1,%d] for %dx%d", l, min_dim, m,
                    n);
    if (q < 0 || s < 1) return fail(ORC_EDIM, "sample_right: q=%d, s=%d out of range", q, s);
    double* om = dalloc((size_t)n * l);
    double* z = dalloc((size_t)n * l);
    orc_gaussian_matrix(n, l, r, om);
    mm(0, 0, a, m, n, om, n, l, y, m, l);
    for (int j = 1; j <= q; ++j) {
        if ((2 * j - 2) % s == 0) orth_inplace(y, m, l);
        mm(1, 0, a, m, n, y, m, l, z, n, l);
        if ((2 * j - 1) % s == 0) orth_inplace(z, n, l);
        mm(0, 0, a, m, n, z, n, l, y, m, l);
    }
    free(om);
    free(z);
    return ORC_OK;
}

/* sketch.hpp:65-67: transpose(sample_right(transpose(A))).  NN on A^T equals
 * TN on A bitwise (same products, same ascending accumulation from 0), so the
 * transposed copy is never formed. y is l x n. */
int orc_sample_left(const double* a, int m, int n, int l, int q, int s, orc_rng* r, double* y) {
    const int min_dim = m < n ? m : n;
    if (l < 1 || l > min_dim)
        return fail(ORC_EDIM, "sample_right: width %d out of range [1,%d] for %dx%d", l, min_dim, n,
                    m);
    if (q < 0 || s < 1) return fail(ORC_EDIM, "sample_right: q=%d, s=%d out of range", q, s);
    double* om = dalloc((size_t)m * l);
    double* y1 = dalloc((size_t)n * l); /* (A^T) * Omega, n x l */
    double* z = dalloc((size_t)m * l);
    orc_gaussian_matrix(m, l, r, om);
    mm(1, 0, a, m, n, om, m, l, y1, n, l);
    for (int j = 1; j <= q; ++j) {
        if ((2 * j - 2) % s == 0) orth_inplace(y1, n, l);
        mm(0, 0, a, m, n, y1, n, l, z, m, l);
        if ((2 * j - 1) % s == 0) orth_inplace(z, m, l);
        mm(1, 0, a, m, n, z, m, l, y1, n, l);
    }
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < l; ++i) y[IDX(i, j, l)] = y1[IDX(j, i, n)];
    free(om);
    free(y1);
    free(z);
    return ORC_OK;
}

/* ------------------------------------------------------------------ rsvd --- */
static int check_sample_rank(int k, int p, int m, int n) {
    if (k < 1) return fail(ORC_EDIM, "rank k must be >= 1 (got %d)", k);
    if (p < 0) return fail(ORC_EDIM, "oversampling p must be >= 0 (got %d)", p);
    const int r = m < n ? m : n;
    if (k + p > r) return fail(ORC_EDIM, "k + p = %d exceeds min(m,n) = %d", k + p, r);
    return ORC_OK;
}

/* rsvd.hpp:144-156 finish_qb_qr_bt: q m x l, bt n x l */
static int finish_qr_bt(const double* q, int m, const double* bt, int n, int l, int k, double* u,
                        double* sigma, double* v) {
    if (k < 1 || k > l) return fail(ORC_EDIM, "rank k = %d outside [1, %d]", k, l);
    double* fq = dalloc((size_t)n * l);
    double* fr = dalloc((size_t)l * l);
    double* ru = dalloc((size_t)l * l);
    double* rs = dalloc((size_t)l);
    double* rv = dalloc((size_t)l * l);
    int st = orc_compact_qr(bt, n, l, fq, fr, NULL);
    if (!st) st = orc_small_svd(fr, l, l, ru, rs, rv);
    if (!st) {
        /* first k columns of Q*Vhat and Qhat*Uhat (column-independent) */
        mm(0, 0, q, m, l, rv, l, k, u, m, k);
        mm(0, 0, fq, n, l, ru, l, k, v, n, k);
        memcpy(sigma, rs, sizeof(double) * (size_t)k);
    }
    free(fq);
    free(fr);
    free(ru);
    free(rs);
    free(rv);
    return st;
}

/* rsvd.hpp:115-140 finish_qb_bbt: q m x l, b l x n (ld ldb) */
static int finish_bbt(const double* q, int m, const double* b, int ldb, int l, int n, int k,
                      double* u, double* sigma, double* v) {
    if (k < 1 || k > l) return fail(ORC_EDIM, "rank k = %d outside [1, %d]", k, l);
    double* bc = dalloc((size_t)l * n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < l; ++i) bc[IDX(i, j, l)] = b[IDX(i, j, ldb)];
    double* t = dalloc((size_t)l * l);
    double* ev = dalloc((size_t)l);
    double* evec = dalloc((size_t)l * l);
    mm(0, 1, bc, l, n, bc, l, n, t, l, l);
    int st = orc_sym_eig(t, l, ev, evec);
    if (!st) {
        const double dmax = ev[0];
        for (int i = 0; i < k && !st; ++i) {
            const double d = ev[i];
            if (d <= 0.0 || d < 1e-28 * dmax)
                st = fail(ORC_ENUM,
                          "rank k exceeds numerical rank for v1; use v2 (eigenvalue %.3e at index "
                          "%d vs max %.3e)",
                          d, i, dmax);
            else
                sigma[i] = sqrt(d);
        }
    }
    if (!st) {
        mm(0, 0, q, m, l, evec, l, k, u, m, k);
        mm(1, 0, bc, l, n, evec, l, k, v, n, k);
        for (int j = 0; j < k; ++j) {
            const double inv = 1.0 / sigma[j];
            for (int i = 0; i < n; ++i) v[IDX(i, j, n)] *= inv;
        }
    }
    free(bc);
    free(t);
    free(ev);
    free(evec);
    return st;
}

/* rsvd.hpp:127-160 */
int orc_rsvd(int variant, const double* a, int m, int n, int k, int p, int q, int s, orc_rng* r,
             double* u, double* sigma, double* v) {
    int st = check_sample_rank(k, p, m, n);
    if (st) return st;
    const int l = k + p;
    double* y = dalloc((size_t)m * l);
    if (variant == 2) {
        /* rsvd_basic: Fig. 1 literally */
        double* g = dalloc((size_t)n * l);
        orc_gaussian_matrix(n, l, r, g);
        mm(0, 0, a, m, n, g, n, l, y, m, l);
        free(g);
        orth_inplace(y, m, l);
        double* b = dalloc((size_t)l * n);
        mm(1, 0, y, m, l, a, m, n, b, l, n);
        const int rr = l < n ? l : n;
        double* bu = dalloc((size_t)l * rr);
        double* bs = dalloc((size_t)rr);
        double* bv = dalloc((size_t)n * rr);
        st = orc_small_svd(b, l, n, bu, bs, bv);
        if (!st) {
            mm(0, 0, y, m, l, bu, l, k, u, m, k);
            memcpy(v, bv, sizeof(double) * (size_t)n * k);
            memcpy(sigma, bs, sizeof(double) * (size_t)k);
        }
        free(b);
        free(bu);
        free(bs);
        free(bv);
        free(y);
        return st;
    }
    st = orc_sample_right(a, m, n, l, q, s, r, y);
    if (!st) st = orth_inplace(y, m, l);
    if (!st) {
        if (variant == 0) {
            double* bt = dalloc((size_t)n * l);
            mm(1, 0, a, m, n, y, m, l, bt, n, l);
            st = finish_qr_bt(y, m, bt, n, l, k, u, sigma, v);
            free(bt);
        } else {
            double* b = dalloc((size_t)l * n);
            mm(1, 0, y, m, l, a, m, n, b, l, n);
            st = finish_bbt(y, m, b, l, l, n, k, u, sigma, v);
            free(b);
        }
    }
    free(y);
    return st;
}

/* ------------------------------------------------------------------- qb --- */
/* qb.hpp:98-152 */
int orc_qb_blocked(const double* a, int m, int n, int blk, int num_blocks, double tol, int q_power,
                   int reorth_period, orc_rng* r, double* Q, double* B, int cap, int* ell_out,
                   double* hist, int* nhist, double* final_resid, int* reached_out, double* w_out) {
    if (blk < 1) return fail(ORC_EDIM, "block size b must be >= 1 (got %d)", blk);
    if (num_blocks < 1) return fail(ORC_EDIM, "block count M must be >= 1 (got %d)", num_blocks);
    if (tol < 0.0) return fail(ORC_EDIM, "tol must be >= 0 (got %g)", tol);
    if (q_power < 0)
        return fail(ORC_EDIM, "power iteration count must be >= 0 (got %d)", q_power);
    if (reorth_period < 1)
        return fail(ORC_EDIM, "reorth_period must be >= 1 (got %d)", reorth_period);
    const int rmax = m < n ? m : n;
    double* w = dalloc((size_t)m * n);
    memcpy(w, a, sizeof(double) * (size_t)m * n);
    double* qi = dalloc((size_t)m * blk);
    double* zi = dalloc((size_t)n * blk);
    double* om = dalloc((size_t)n * blk);
    double* proj = dalloc((size_t)(cap > 0 ? cap : 1) * blk);
    double* tmp = dalloc((size_t)m * blk);
    double* bi = dalloc((size_t)blk * n);
    double* col = dalloc((size_t)m);
    int ell = 0, nh = 0, reached = 0;
    double resid = orc_frobenius(w, (int64_t)m * n);
    for (int i = 1; i <= num_blocks; ++i) {
        int width = blk < rmax - ell ? blk : rmax - ell;
        if (width < 1) break;
        orc_rng br;
        orc_rng_substream(r, &br);
        orc_gaussian_matrix(n, width, &br, om);
        mm(0, 0, w, m, n, om, n, width, qi, m, width);
        orth_inplace(qi, m, width);
        for (int j = 0; j < q_power; ++j) {
            mm(1, 0, w, m, n, qi, m, width, zi, n, width);
            orth_inplace(zi, n, width);
            mm(0, 0, w, m, n, zi, n, width, qi, m, width);
            orth_inplace(qi, m, width);
        }
        if (i % reorth_period == 0) {
            if (ell > 0) {
                mm(1, 0, Q, m, ell, qi, m, width, proj, ell, width);
                mm(0, 0, Q, m, ell, proj, ell, width, tmp, m, width);
                for (size_t t = 0; t < (size_t)m * width; ++t) qi[t] = qi[t] - tmp[t];
            }
            orth_inplace(qi, m, width);
        }
        mm(1, 0, qi, m, width, w, m, n, bi, width, n);
        memcpy(Q + IDX(0, ell, m), qi, sizeof(double) * (size_t)m * width);
        for (int j = 0; j < n; ++j)
            for (int t = 0; t < width; ++t) B[IDX(ell + t, j, cap)] = bi[IDX(t, j, width)];
        ell += width;
        /* w = w - qi*bi, one column of the product at a time */
        for (int j = 0; j < n; ++j) {
            mm(0, 0, qi, m, width, bi + IDX(0, j, width), width, 1, col, m, 1);
            double* wj = w + IDX(0, j, m);
            for (int t = 0; t < m; ++t) wj[t] = wj[t] - col[t];
        }
        resid = orc_frobenius(w, (int64_t)m * n);
        hist[nh++] = resid;
        if (tol > 0.0 && resid < tol) {
            reached = 1;
            break;
        }
    }
    *ell_out = ell;
    *nhist = nh;
    *final_resid = resid;
    *reached_out = tol > 0.0 ? reached : 1;
    if (w_out) memcpy(w_out, w, sizeof(double) * (size_t)m * n);
    free(w);
    free(qi);
    free(zi);
    free(om);
    free(proj);
    free(tmp);
    free(bi);
    free(col);
    return ORC_OK;
}

/* qb.hpp:276-288 */
int orc_svd_from_qb(const double* q, const double* b, int ldb, int m, int n, int ell, int k,
                    int vnum, double* u, double* sigma, double* v, int* k_out) {
    if (k < 0 || k > ell) return fail(ORC_EDIM, "rank k = %d outside [0, rank(B) = %d]", k, ell);
    if (k == 0) k = ell;
    *k_out = k;
    if (k == 0) return ORC_OK;
    if (vnum == 1) return finish_bbt(q, m, b, ldb, ell, n, k, u, sigma, v);
    double* bt = dalloc((size_t)n * ell);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < ell; ++i) bt[IDX(j, i, n)] = b[IDX(i, j, ldb)];
    int st = finish_qr_bt(q, m, bt, n, ell, k, u, sigma, v);
    free(bt);
    return st;
}

/* ---------------------------------------------------------------- interp --- */
/* interp.hpp:65-72 */
static void build_interp(const int* perm, const double* t, int ldt, int n, int k, double* v) {
    memset(v, 0, sizeof(double) * (size_t)n * k);
    for (int i = 0; i < k; ++i) v[IDX(perm[i], i, n)] = 1.0;
    for (int c = 0; c + k < n; ++c)
        for (int j = 0; j < k; ++j) v[IDX(perm[k + c], j, n)] = t[IDX(j, c, ldt)];
}

/* interp.hpp:74-117 id_column (also id_row through the transpose) */
int orc_id_column(const double* a, int m, int n, int k, double tol, int* jc, double* v,
                  int* k_out, double* qr_residual, int* reached, int* clamped) {
    const int rmax = m < n ? m : n;
    const int tol_mode = (k == 0 && tol > 0.0);
    const int kmax = tol_mode ? rmax : (k > 0 ? k : 1);
    double* q1 = dalloc((size_t)m * kmax);
    double* s1 = dalloc((size_t)kmax * n);
    int frank = 0, deg = 0, rch = 0;
    double res = 0.0;
    int st = orc_pivoted_qr(a, m, n, k, tol, q1, s1, kmax, jc, &frank, &res, &rch, &deg);
    if (st) {
        free(q1);
        free(s1);
        return st;
    }
    *k_out = frank;
    *qr_residual = res;
    *reached = tol > 0.0 ? rch : 1;
    *clamped = 0;
    if (frank > 0) {
        double* t = dalloc((size_t)frank * (n > frank ? n - frank : 1));
        if (n > frank)
            st = orc_upper_tri_solve(s1, kmax, frank, s1 + IDX(0, frank, kmax), kmax, n - frank, t,
                                     clamped);
        if (!st) build_interp(jc, t, frank, n, frank, v);
        free(t);
    }
    free(q1);
    free(s1);
    return st;
}

/* interp.hpp:203-223 */
int orc_id_rand(const double* a, int m, int n, int k, int p, int q, int s, orc_rng* r, int* jc,
                double* v, double* qr_residual, int* clamped) {
    if (k < 1) return fail(ORC_EDIM, "rank k must be >= 1 (got %d)", k);
    if (p < 0) return fail(ORC_EDIM, "oversampling p must be >= 0 (got %d)", p);
    if (k + p > (m < n ? m : n))
        return fail(ORC_EDIM, "k + p = %d exceeds min(m,n) = %d", k + p, m < n ? m : n);
    const int l = k + p;
    double* y = dalloc((size_t)l * n);
    int st = orc_sample_left(a, m, n, l, q, s, r, y);
    if (st) {
        free(y);
        return st;
    }
    double* q1 = dalloc((size_t)l * l);
    double* s1 = dalloc((size_t)l * n);
    int frank, rch, deg;
    double res;
    st = orc_pivoted_qr(y, l, n, l, 0.0, q1, s1, l, jc, &frank, &res, &rch, &deg);
    if (!st) {
        /* frobenius_norm(submatrix(s1, k, l-k, k, n-k)): one Kahan pass */
        double sum = 0.0, comp = 0.0;
        for (int j = k; j < n; ++j)
            for (int i = k; i < l; ++i) {
                const double x = s1[IDX(i, j, l)];
                const double term = x * x;
                const double yy = term - comp;
                const double t = sum + yy;
                comp = (t - sum) - yy;
                sum = t;
            }
        *qr_residual = sqrt(sum);
        *clamped = 0;
        double* t = dalloc((size_t)k * (n > k ? n - k : 1));
        if (n > k) st = orc_upper_tri_solve(s1, l, k, s1 + IDX(0, k, l), l, n - k, t, clamped);
        if (!st) build_interp(jc, t, k, n, k, v);
        free(t);
    }
    free(y);
    free(q1);
    free(s1);
    return st;
}

/* interp.hpp:123-140 */
int orc_two_sided_from_column(const double* a, int m, int n, const int* jc, int k, int* jr,
                              double* w) {
    (void)n;
    if (k == 0) {
        for (int i = 0; i < m; ++i) jr[i] = i;
        return ORC_OK;
    }
    /* C^T (k x m) straight from A's skeleton columns */
    double* ct = dalloc((size_t)k * m);
    for (int j = 0; j < k; ++j)
        for (int i = 0; i < m; ++i) ct[IDX(j, i, k)] = a[IDX(i, jc[j], m)];
    int kk, rch, cl;
    double res;
    int st = orc_id_column(ct, k, m, k, 0.0, jr, w, &kk, &res, &rch, &cl);
    free(ct);
    return st;
}

/* interp.hpp:143-177 */
int orc_cur_from_two_sided(const double* a, int m, int n, const int* jc, const int* jr,
                           const double* v, int k, double* c, double* u, double* r,
                           double* residual) {
    if (k == 0) {
        *residual = orc_frobenius(a, (int64_t)m * n);
        return ORC_OK;
    }
    for (int j = 0; j < k; ++j) memcpy(c + IDX(0, j, m), a + IDX(0, jc[j], m), sizeof(double) * m);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < k; ++i) r[IDX(i, j, k)] = a[IDX(jr[i], j, m)];
    /* cur_linkage: compact_qr(R^T) */
    double* rt = dalloc((size_t)n * k);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < k; ++i) rt[IDX(j, i, n)] = r[IDX(i, j, k)];
    double* fq = dalloc((size_t)n * k);
    double* fr = dalloc((size_t)k * k);
    int st = orc_compact_qr(rt, n, k, fq, fr, NULL);
    if (!st) {
        double dmax = 0.0;
        for (int i = 0; i < k; ++i)
            if (fabs(fr[IDX(i, i, k)]) > dmax) dmax = fabs(fr[IDX(i, i, k)]);
        for (int i = 0; i < k && !st; ++i)
            if (dmax == 0.0 || fabs(fr[IDX(i, i, k)]) < 1e-13 * dmax)
                st = fail(ORC_ENUM,
                          "CUR linkage: skeleton row %d makes R rank-deficient to working precision",
                          jr[i]);
    }
    if (!st) {
        double* qtv = dalloc((size_t)k * k);
        double* t = dalloc((size_t)k * k);
        int cl;
        mm(1, 0, fq, n, k, v, n, k, qtv, k, k);
        st = orc_upper_tri_solve(fr, k, k, qtv, k, k, t, &cl);
        if (!st) {
            for (int j = 0; j < k; ++j)
                for (int i = 0; i < k; ++i) u[IDX(i, j, k)] = t[IDX(j, i, k)];
            double* ur = dalloc((size_t)k * n);
            double* cur = dalloc((size_t)m * n);
            mm(0, 0, u, k, k, r, k, n, ur, k, n);
            mm(0, 0, c, m, k, ur, k, n, cur, m, n);
            for (size_t t2 = 0; t2 < (size_t)m * n; ++t2) cur[t2] = a[t2] - cur[t2];
            *residual = orc_frobenius(cur, (int64_t)m * n);
            free(ur);
            free(cur);
        }
        free(qtv);
        free(t);
    }
    free(rt);
    free(fq);
    free(fr);
    return st;
}

/* interp.hpp:240-244 */
int orc_cur_rand(const double* a, int m, int n, int k, int p, int q, int s, orc_rng* rng, int* jc,
                 int* jr, double* v, double* w, double* c, double* u, double* r,
                 double* residual, double* qr_residual) {
    int clamped;
    int st = orc_id_rand(a, m, n, k, p, q, s, rng, jc, v, qr_residual, &clamped);
    if (!st) st = orc_two_sided_from_column(a, m, n, jc, k, jr, w);
    if (!st) st = orc_cur_from_two_sided(a, m, n, jc, jr, v, k, c, u, r, residual);
    return st;
}

/* interp.hpp:228-236 (shape checks live with the caller) */
int orc_id_from_qb(const double* b, int ldb, int ell, int n, int k, int* jc, double* v,
                   double* qr_residual, int* clamped) {
    if (k < 1 || k > ell) return fail(ORC_EDIM, "rank k = %d outside [1, rank(B) = %d]", k, ell);
    double* bc = dalloc((size_t)ell * n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < ell; ++i) bc[IDX(i, j, ell)] = b[IDX(i, j, ldb)];
    int kk, rch;
    int st = orc_id_column(bc, ell, n, k, 0.0, jc, v, &kk, qr_residual, &rch, clamped);
    free(bc);
    return st;
}
