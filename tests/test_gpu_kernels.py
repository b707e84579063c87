"""Kernel-level parity: the CUDA engine against the CPU oracle (oracle/,
bit-identical to the reference) on the same seeded inputs.  Tolerances are the
reference's own test tolerances (tests/test_matmul.cpp:30-56,
tests/test_qr.cpp:32-64, tests/test_jacobi.cpp:110-142)."""
import numpy as np
import pytest

import paper_1502_05366_b200 as R
from helpers import exact_rank, match_columns_up_to_sign, orthonormality_defect, rel_fro

ROOT = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("m,n,k", [(5, 3, 4), (37, 29, 53), (130, 70, 300), (257, 190, 1000),
                                   (1001, 211, 777)])
def test_matmul_four_cases_vs_oracle(eng, orc, ta, tb, m, n, k):
    rs = np.random.default_rng(m * 7 + n + k + 3 * ta + tb)
    a = rs.standard_normal((k, m) if ta else (m, k))
    b = rs.standard_normal((n, k) if tb else (k, n))
    got = eng.matmul(a, b, bool(ta), bool(tb))
    want = orc.matmul(a, b, ta, tb)
    assert got.shape == want.shape
    assert rel_fro(got, want) <= 1e-13  # test_matmul.cpp:30-39


def test_matmul_hand_arithmetic(eng):
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    b = np.array([[5.0, 6.0], [7.0, 8.0]])
    np.testing.assert_array_equal(eng.matmul(a, b), np.array([[19.0, 22.0], [43.0, 50.0]]))


def test_matmul_shape_error_names_both_shapes(eng):
    with pytest.raises(R.DimensionError) as e:
        eng.matmul(np.zeros((3, 4)), np.zeros((5, 2)))
    assert "3x4" in str(e.value) and "5x2" in str(e.value)


def test_matmul_bitwise_deterministic(eng):
    rs = np.random.default_rng(5)
    a = rs.standard_normal((3000, 700))
    b = rs.standard_normal((700, 300))
    x = eng.matmul(a, b)
    for _ in range(3):
        assert np.array_equal(eng.matmul(a, b), x)
    c = rs.standard_normal((3000, 300))
    y = eng.matmul(a, c, True, False)  # split-K path: deterministic reduction order
    for _ in range(3):
        assert np.array_equal(eng.matmul(a, c, True, False), y)


def test_orth_kat_and_conventions(eng):
    q = eng.orth(np.array([[3.0], [4.0]]))
    assert abs(q[0, 0] - 0.6) <= 1e-15 and abs(q[1, 0] - 0.8) <= 1e-15  # test_qr.cpp:14-20


@pytest.mark.parametrize("m,n", [(50, 8), (40, 10), (2000, 210), (5000, 300)])
def test_compact_qr_vs_oracle(eng, orc, m, n):
    rs = np.random.default_rng(m + n)
    a = rs.standard_normal((m, n))
    q, r, deg = eng.compact_qr(a)
    qo, ro, _ = orc.compact_qr(a)
    assert not deg
    assert orthonormality_defect(q) <= 1e-13 * np.sqrt(n)
    assert rel_fro(q @ r, a) <= 1e-13
    assert np.all(np.diag(r) >= 0) and np.all(np.tril(r, -1) == 0)
    assert rel_fro(q, qo) <= 1e-12  # diag(R) >= 0 makes Q unique
    assert rel_fro(r, ro) <= 1e-12


def test_compact_qr_exact_dependence_and_zero_column(eng):
    rs = np.random.default_rng(24)
    c = rs.standard_normal((30, 1))
    a = np.hstack([c, c])
    _, r, _ = eng.compact_qr(a)
    assert abs(r[1, 1]) <= 1e-12 * np.linalg.norm(a)  # test_qr.cpp:66-72
    c = rs.standard_normal((6, 1))
    a = np.hstack([c, np.zeros((6, 1))])
    q, r, deg = eng.compact_qr(a)
    assert deg and r[1, 1] == 0.0  # test_qr.cpp:74-83
    assert orthonormality_defect(q) <= 1e-13


def test_compact_qr_upper_triangular_fixed_point(eng):
    a = np.array([[2.0, 1.0, 0.5], [0.0, 3.0, 1.5], [0.0, 0.0, 1.0]])
    q, r, _ = eng.compact_qr(a)
    assert np.max(np.abs(q - np.eye(3))) <= 1e-14
    assert np.max(np.abs(r - a)) <= 1e-14


def test_compact_qr_rank_deficient_tall_falls_back(eng):
    a = exact_rank(400, 60, 7, 3)
    q, r, _ = eng.compact_qr(a)
    assert orthonormality_defect(q) <= 1e-12
    assert rel_fro(q @ r, a) <= 1e-13


def test_orth_rejects_wide(eng):
    with pytest.raises(R.DimensionError):
        eng.orth(np.zeros((3, 5)))


@pytest.mark.parametrize("m,n,k", [(60, 40, 15), (35, 50, 20), (50, 30, 25), (610, 3000, 610), (900, 1500, 300),
                                   (200, 30000, 50)])
def test_pivoted_qr_vs_oracle(eng, orc, m, n, k):
    """(900, 1500): trailing columns longer than the register tile take the
    loop form for the first steps; (200, 30000): the position maps do not fit
    shared memory, so the two-barrier kernel runs."""
    rs = np.random.default_rng(m * 3 + n)
    a = rs.standard_normal((m, n))
    got = eng.pivoted_qr_partial(a, k)
    want = orc.pivoted_qr(a, k)
    assert got["frank"] == want["frank"] == k
    np.testing.assert_array_equal(got["perm"], want["perm"])
    assert rel_fro(got["s1"], want["s1"]) <= 1e-11
    assert abs(got["residual"] - want["residual"]) <= 1e-10 * max(1.0, want["residual"])
    assert rel_fro(got["q1"], want["q1"]) <= 1e-11


def test_pivoted_qr_kats(eng):
    f = eng.pivoted_qr_partial(np.diag([3.0, 2.0, 1.0]), 2)
    assert f["frank"] == 2 and list(f["perm"][:2]) == [0, 1]
    assert abs(f["residual"] - 1.0) <= 1e-14  # test_qr.cpp:85-92
    rs = np.random.default_rng(26)
    a = rs.standard_normal((20, 2)) @ rs.standard_normal((20, 2)).T
    f = eng.pivoted_qr_partial(a, 0, 1e-10)
    assert f["frank"] == 2 and f["tolerance_reached"]  # :94-102
    f = eng.pivoted_qr_partial(rs.standard_normal((12, 12)), 0, 1e-20)
    assert f["frank"] == 12 and not f["tolerance_reached"] and f["residual"] > 1e-20
    for k, tol in [(2, 1e-3), (0, 0.0), (5, 0.0)]:
        with pytest.raises(R.DimensionError):
            eng.pivoted_qr_partial(np.zeros((4, 4)), k, tol)


def test_pivoted_qr_tol_mode_vs_oracle(eng, orc):
    rs = np.random.default_rng(77)
    a = rs.standard_normal((40, 6)) @ np.diag(np.logspace(0, -6, 6)) @ rs.standard_normal((6, 30))
    got = eng.pivoted_qr_partial(a, 0, 1e-4)
    want = orc.pivoted_qr(a, 0, 1e-4)
    assert got["frank"] == want["frank"]
    np.testing.assert_array_equal(got["perm"][: got["frank"]], want["perm"][: want["frank"]])
    assert got["tolerance_reached"] == want["reached"]


def test_upper_tri_solve(eng, orc):
    t, cl = eng.upper_tri_solve(np.array([[2.0, 1.0], [0.0, 1.0]]), np.array([[3.0], [1.0]]))
    assert not cl and np.allclose(t, [[1.0], [1.0]], atol=1e-15)
    t, cl = eng.upper_tri_solve(np.eye(3), np.arange(6.0).reshape(3, 2))
    assert np.array_equal(t, np.arange(6.0).reshape(3, 2)) and not cl
    t, cl = eng.upper_tri_solve(np.array([[1e8, 0.0], [0.0, 1e-8]]), np.array([[1.0], [1.0]]))
    assert cl and abs(t[0, 0] - 1e-8) <= 1e-20 and t[1, 0] == 1e4  # test_qr.cpp:203-219
    t, cl = eng.upper_tri_solve(np.eye(2), np.array([[1e5], [2e5]]))
    assert not cl and t[1, 0] == 2e5
    with pytest.raises(R.NumericalError):
        eng.upper_tri_solve(np.array([[1.0, 2.0], [0.0, 0.0]]), np.ones((2, 1)))
    rs = np.random.default_rng(30)
    s11 = np.triu(rs.standard_normal((600, 600))) + 30 * np.eye(600)
    s12 = rs.standard_normal((600, 900))
    got, _ = eng.upper_tri_solve(s11, s12)
    want, _ = orc.upper_tri_solve(s11, s12)
    assert rel_fro(got, want) <= 1e-12


@pytest.mark.parametrize("k,nc", [(1, 5), (64, 3), (65, 70), (2001, 1500)])
def test_upper_tri_solve_blocked_vs_oracle(eng, orc, k, nc):
    """The blocked DMMA back substitution (64-row diagonal blocks, GEMM
    updates; no shared-memory bound on k) against the oracle's
    row-oriented substitution (core/qr.hpp:242-275), ragged last blocks
    included; a graded, well-conditioned S11 so only rounding differs."""
    rs = np.random.default_rng(k + nc)
    s11 = np.triu(rs.standard_normal((k, k)), 1) * (0.5 / np.sqrt(k)) + np.diag(np.linspace(2.0, 0.5, k))
    s12 = rs.standard_normal((k, nc))
    got, cl = eng.upper_tri_solve(s11, s12)
    want, clo = orc.upper_tri_solve(s11, s12)
    assert cl == clo
    assert rel_fro(got, want) <= 1e-10


@pytest.mark.parametrize("m,n", [(40, 40), (60, 25), (25, 60), (210, 210), (510, 510), (3, 1), (1, 3)])
def test_small_svd_vs_oracle(eng, orc, m, n):
    rs = np.random.default_rng(m * 11 + n)
    a = rs.standard_normal((m, n))
    u, s, v = eng.small_svd(a)
    uo, so, vo = orc.small_svd(a)
    r = min(m, n)
    assert u.shape == (m, r) and v.shape == (n, r)
    assert np.all(np.diff(s) <= 0)
    assert np.max(np.abs(s - so) / so[0]) <= 1e-13
    assert rel_fro((u * s) @ v.T, a) <= 1e-12  # test_jacobi.cpp:110-142
    assert orthonormality_defect(u) <= 1e-11 and orthonormality_defect(v) <= 1e-11
    assert match_columns_up_to_sign(u, uo) <= 1e-8


@pytest.mark.parametrize("m,n,decay", [(2000, 120, 0.0), (1800, 200, 30.0)])
def test_small_svd_gram_block_jacobi_vs_oracle(eng, orc, m, n, decay):
    """Columns too long for shared memory (16 x m doubles > 200 KB) take the
    Gram block Jacobi kernel: same sigma as the reference's one-sided sweep
    (graded spectra included), orthonormal factors, reconstruction."""
    rs = np.random.default_rng(m + n)
    a = rs.standard_normal((m, n))
    if decay:
        q1, _ = np.linalg.qr(rs.standard_normal((m, n)))
        q2, _ = np.linalg.qr(rs.standard_normal((n, n)))
        a = (q1 * np.exp(-np.arange(n) / decay)) @ q2.T
    u, s, v = eng.small_svd(a)
    uo, so, vo = orc.small_svd(a)
    assert np.all(np.diff(s) <= 0)
    assert np.max(np.abs(s - so) / so) <= 1e-10
    assert rel_fro((u * s) @ v.T, a) <= 1e-12
    assert orthonormality_defect(u) <= 1e-11 and orthonormality_defect(v) <= 1e-11


@pytest.mark.parametrize("m,n,kind", [(1300, 1000, "graded"), (700, 37, "gauss"), (520, 17, "gauss"),
                                      (300, 100, "deficient"), (400, 96, "scaled"), (64, 64, "gauss")])
def test_small_svd_shared_gram_jacobi_vs_oracle(eng, orc, m, n, kind):
    """The shared-memory-resident Gram block Jacobi (l <= ~1400; blocks of 16
    columns when the pair fits, else 8): ragged last blocks, zero and repeated
    columns (completion), columns scaled over 60 decades, graded spectra —
    the reference's sigma, orthonormal factors, reconstruction."""
    rs = np.random.default_rng(m * 7 + n)
    a = rs.standard_normal((m, n))
    if kind == "graded":
        q1, _ = np.linalg.qr(rs.standard_normal((m, n)))
        q2, _ = np.linalg.qr(rs.standard_normal((n, n)))
        a = (q1 * np.exp(-np.arange(n) / 100.0)) @ q2.T
    elif kind == "deficient":
        a[:, 10:20] = 0.0
        a[:, 30:40] = a[:, 50:60]
    elif kind == "scaled":
        a = a * 10.0 ** (-np.arange(n) * 60.0 / n)
    u, s, v = eng.small_svd(a)
    uo, so, vo = orc.small_svd(a)
    r = min(m, n)
    assert u.shape == (m, r) and v.shape == (n, r)
    assert np.all(np.diff(s) <= 0)
    if kind == "deficient":
        nz = so > 1e-10 * so[0]
        assert np.max(np.abs(s[nz] - so[nz]) / so[nz]) <= 1e-11
        assert np.all(s[~nz] <= 1e-12 * so[0])
    else:
        assert np.max(np.abs(s - so) / so) <= 1e-10
    assert rel_fro((u * s) @ v.T, a) <= 1e-12
    assert orthonormality_defect(u) <= 1e-11 and orthonormality_defect(v) <= 1e-11


@pytest.mark.parametrize("env", [{"RLRA_BGRAM_NOHELP": "1"}, {"RLRA_SVD_KERNEL": "block"},
                                 {"RLRA_BGRAM_BW": "16"}, {"RLRA_SVD_KERNEL": "gram"},
                                 {"RLRA_SVD_KERNEL": "sgram"}])
def test_small_svd_variants_agree(eng, env):
    """The Jacobi variants selectable by environment (bgram without V
    helpers, 16-column blocks, the one-sided block kernel, the 32-column
    streaming kernel) give the default path's sigma and reconstruction."""
    import json
    import os
    import subprocess
    import sys

    rs = np.random.default_rng(5)
    a = rs.standard_normal((600, 400)) * np.exp(-np.arange(400) / 60.0)
    u, s, v = eng.small_svd(a)
    code = ("import sys, json, numpy as np; sys.path.insert(0, %r); import paper_1502_05366_b200 as R; "
            "a = np.random.default_rng(5).standard_normal((600, 400)) * np.exp(-np.arange(400) / 60.0); "
            "u, s, v = R.Engine(0).small_svd(a); print(json.dumps(s.tolist()))" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr
    s2 = np.array(json.loads(out.stdout.strip().splitlines()[-1]))
    assert np.max(np.abs(s2 - s) / s) <= 1e-12
    assert rel_fro((u * s) @ v.T, a) <= 1e-12


@pytest.mark.parametrize("m,n,kind", [(256, 256, "graded"), (210, 210, "graded"), (300, 100, "deficient"),
                                      (520, 17, "gauss"), (130, 129, "scaled"), (250, 250, "gauss")])
def test_small_svd_cluster_kernel_bit_identical(eng, tmp_path, m, n, kind):
    """l <= 256 runs the cluster-resident kernel (W in shared memory, st.async
    exchange, V replayed from the rotation log); it performs the L2 variant's
    arithmetic in the same order, so U, sigma and V are bit-identical to
    RLRA_SVD_KERNEL=bgram's (a separate process: the choice is read once)."""
    import os
    import subprocess
    import sys

    rs = np.random.default_rng(m * 13 + n)
    a = rs.standard_normal((m, n))
    if kind == "graded":
        q1, _ = np.linalg.qr(rs.standard_normal((m, n)))
        q2, _ = np.linalg.qr(rs.standard_normal((n, n)))
        a = (q1 * np.exp(-np.arange(n) / 20.0)) @ q2.T
    elif kind == "deficient":
        a[:, 10:20] = 0.0
        a[:, 30:40] = a[:, 50:60]
    elif kind == "scaled":
        a = a * 10.0 ** (-np.arange(n) * 30.0 / n)
    np.save(tmp_path / "a.npy", a)
    u, s, v = eng.small_svd(a)
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_1502_05366_b200 as R; "
            "a = np.load(%r); u, s, v = R.Engine(0).small_svd(a); np.savez(%r, u=u, s=s, v=v)"
            % (ROOT, str(tmp_path / "a.npy"), str(tmp_path / "b.npz")))
    out = subprocess.run([sys.executable, "-c", code], env={**os.environ, "RLRA_SVD_KERNEL": "bgram"},
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    b = np.load(tmp_path / "b.npz")
    assert np.array_equal(s, b["s"]) and np.array_equal(u, b["u"]) and np.array_equal(v, b["v"])
    assert orthonormality_defect(u) <= 1e-11 and orthonormality_defect(v) <= 1e-11


def test_small_svd_kats(eng):
    _, s, _ = eng.small_svd(np.diag([2.0, -3.0]))
    assert np.allclose(s, [3.0, 2.0], rtol=1e-15)  # test_jacobi.cpp:95-101
    a = np.zeros((5, 3))
    a[:, 0] = [1, 2, 3, 4, 5]
    u, s, v = eng.small_svd(a)
    assert s[1] == 0.0 and s[2] == 0.0
    assert orthonormality_defect(u) <= 1e-13  # completion (test_jacobi.cpp:154-163)


@pytest.mark.parametrize("n", [2, 7, 40, 211])
def test_sym_eig_vs_oracle(eng, orc, n):
    rs = np.random.default_rng(n)
    b = rs.standard_normal((n, n))
    t = b @ b.T
    d, e = eng.sym_eig(t)
    do, eo = orc.sym_eig(t)
    assert np.all(np.diff(d) <= 0)
    assert np.max(np.abs(d - do)) <= 1e-12 * abs(do[0])
    assert rel_fro(e @ np.diag(d) @ e.T, t) <= 1e-12


def test_sym_eig_rejects_asymmetry(eng):
    with pytest.raises(R.NumericalError):
        eng.sym_eig(np.array([[1.0, 2.0], [0.0, 1.0]]))


def test_frobenius_norm(eng):
    rs = np.random.default_rng(9)
    a = rs.standard_normal((1234, 567))
    assert abs(eng.frobenius_norm(a) - np.linalg.norm(a)) <= 1e-13 * np.linalg.norm(a)


def test_philox_omega_is_gaussian_and_deterministic(eng):
    g = eng.gaussian_philox(4000, 64, seed=12345)
    assert np.array_equal(g, eng.gaussian_philox(4000, 64, seed=12345))
    assert abs(g.mean()) < 0.01 and abs(g.std() - 1.0) < 0.01
    # row offset addresses the same global stream
    h = eng.gaussian_philox(1000, 64, seed=12345, row0=1000)
    assert np.array_equal(h, g[1000:2000])
    assert not np.array_equal(eng.gaussian_philox(100, 8, seed=1), eng.gaussian_philox(100, 8, seed=2))


@pytest.mark.parametrize("ta", [0, 1])
@pytest.mark.parametrize("m,n,k", [(2048, 200, 700), (2008, 130, 333), (4096, 510, 1500)])
def test_matmul_tma_paths_vs_oracle(eng, orc, ta, m, n, k):
    """The TMA-staged GEMM (gemm_tma.cuh): x-contiguous A as one 3-D box per
    stage (M % 16 == 0) or eight 2-D boxes (M % 16 != 0), k-contiguous A^T,
    split-K for the tall TN shapes; swizzled tiles and permuted fragment rows
    must land every C element where the oracle puts it."""
    rs = np.random.default_rng(m + n + k + ta)
    a = rs.standard_normal((k, m) if ta else (m, k))
    b = rs.standard_normal((k, n))
    got = eng.matmul(a, b, bool(ta), False)
    assert rel_fro(got, orc.matmul(a, b, ta, 0)) <= 1e-13


@pytest.mark.parametrize("ta", [0, 1])
def test_matmul_tail_wave_split_vs_oracle(eng, orc, ta):
    """150 tiles on 148 SMs: the 2 tail tiles run as 8 k-chunks each
    (gemm.cu tail split) and are reduced with alpha/beta afterwards."""
    rs = np.random.default_rng(5 + ta)
    m, n, k = 19200, 100, 1500
    a = rs.standard_normal((k, m) if ta else (m, k))
    b = rs.standard_normal((k, n))
    got = eng.matmul(a, b, bool(ta), False)
    assert rel_fro(got, orc.matmul(a, b, ta, 0)) <= 1e-13


def test_sketch_philox_in_register_equals_materialized(eng):
    """The sketch (Philox Omega materialised by rlra_gaussian_philox, then the
    streaming GEMM) equals A times the same materialised Omega, and the
    in-GEMM generation (RLRA_SKETCH_FUSED=1: producer warps + 2-CTA cluster
    sharing) produces the same bits."""
    import json
    import os
    import subprocess
    import sys

    rs = np.random.default_rng(11)
    m, n, l = 2048, 1000, 130
    a = rs.standard_normal((m, n))
    y = eng.sample_right(a, l, 0, 1, omega=R.Omega.philox(777))
    om = eng.gaussian_philox(n, l, seed=777)
    assert np.array_equal(y, eng.matmul(a, om))
    code = ("import sys, json, numpy as np; sys.path.insert(0, %r); import paper_1502_05366_b200 as R; "
            "a = np.random.default_rng(11).standard_normal((2048, 1000)); "
            "y = R.Engine(0).sample_right(a, 130, 0, 1, omega=R.Omega.philox(777)); "
            "print(json.dumps(y.ravel(order='F').tolist()))" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], env={**os.environ, "RLRA_SKETCH_FUSED": "1"},
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    yf = np.array(json.loads(out.stdout.strip().splitlines()[-1])).reshape((m, l), order="F")
    assert np.array_equal(yf, y)


@pytest.mark.parametrize("n", [1, 5, 64, 65, 200, 510, 1024, 1100])
def test_chol_inv_one_launch_and_blocked(eng, n):
    """CholQR's Cholesky + triangular inverse: the one-launch cooperative
    kernel (n <= 1024) and the launch-per-block GEMM path (n > 1024) against
    numpy's Cholesky of a well-conditioned Gram."""
    rs = np.random.default_rng(n)
    y = rs.standard_normal((3 * n + 10, n))
    g = y.T @ y
    g_in = np.triu(g) + np.tril(rs.standard_normal((n, n)), -1)  # lower triangle is never read
    r, ri, ok = eng.chol_inv(g_in, 1e-12)
    assert ok
    assert np.array_equal(np.tril(r, -1), np.zeros((n, n)))
    assert np.array_equal(np.tril(ri, -1), np.zeros((n, n)))
    want = np.linalg.cholesky(g).T
    assert np.linalg.norm(r - want) <= 1e-12 * np.linalg.norm(want)
    assert np.linalg.norm(ri @ r - np.eye(n)) <= 1e-12 * np.sqrt(n)


def test_chol_inv_flags_rank_deficiency(eng):
    rs = np.random.default_rng(3)
    y = rs.standard_normal((300, 100))
    y[:, 70] = y[:, 3] + y[:, 9]  # exactly dependent column: pivot 70 collapses
    _, _, ok = eng.chol_inv(y.T @ y, 1e-12)
    assert not ok
    _, _, ok = eng.chol_inv(-np.eye(4), 0.0)  # non-positive pivot
    assert not ok


def test_upper_tri_solve_k_beyond_the_old_shared_memory_bound(eng):
    """k = 30000 > the round-1 kernel's ~29k shared-memory cap:
    the blocked solve has no bound on k.  Device buffers through the C-ABI;
    S11 = diag(1..2) + a small strictly upper part, X known, S12 = S11 X."""
    import ctypes as C

    import torch

    k, nc = 30000, 16
    g = torch.Generator(device="cuda").manual_seed(3)
    S = torch.triu(torch.randn(k, k, device="cuda", dtype=torch.float64, generator=g), 1) * (0.3 / k ** 0.5)
    S += torch.diag(torch.linspace(1.0, 2.0, k, device="cuda", dtype=torch.float64))
    X = torch.randn(k, nc, device="cuda", dtype=torch.float64, generator=g)
    B = S @ X
    S_c, B_c = S.t().contiguous(), B.t().contiguous()  # column-major storage
    T = torch.empty(nc, k, device="cuda", dtype=torch.float64)
    torch.cuda.synchronize()  # the engine runs on its own stream
    cl = C.c_int(0)
    st = R.lib().rlra_upper_tri_solve(eng._ctx, R.DEVICE, C.c_void_p(S_c.data_ptr()), k, C.c_int64(k),
                                      C.c_void_p(B_c.data_ptr()), nc, C.c_int64(k), C.c_void_p(T.data_ptr()),
                                      C.c_int64(k), C.byref(cl))
    assert st == 0, R.lib().rlra_last_error()
    err = torch.linalg.norm(T.t() - X) / torch.linalg.norm(X)
    assert float(err) <= 1e-12 and cl.value == 0


@pytest.mark.parametrize("n", [1025, 1500, 2100])
def test_chol_inv_large_blocked_vs_numpy(eng, n):
    """n > 1024: diagonal blocks of 512 by the cooperative kernel, trailing
    updates and the off-diagonal blocks of R^{-1} on the GEMM; R upper with
    R^T R = G, R R^{-1} = I; a rank-deficient Gram is reported as breakdown."""
    rs = np.random.default_rng(n)
    y = rs.standard_normal((2 * n, n)) * np.exp(-np.arange(n) / (n / 6.0))
    g = y.T @ y
    r, ri, ok = eng.chol_inv(g, 1e-12)
    assert ok
    assert np.allclose(np.tril(r, -1), 0.0)
    assert np.linalg.norm(r.T @ r - g) <= 1e-13 * np.linalg.norm(g)
    assert np.linalg.norm(r @ ri - np.eye(n)) <= 1e-9
    yd = y[:, : n // 2]
    gd = np.zeros((n, n))
    gd[: n // 2, : n // 2] = yd.T @ yd  # exactly singular beyond n/2
    _, _, ok2 = eng.chol_inv(gd, 1e-12)
    assert not ok2


@pytest.mark.parametrize("kind,k", [("graded", 120), ("exact_rank", 120), ("graded", 290), ("exact_rank", 290)])
def test_rhat_jacobi_v_from_solve(orc, tmp_path, kind, k):
    """finish_qr_bt's R-hat on the streaming Jacobi (forced here at l = 130
    and l = 300): the sweeps rotate W only and V comes from R^{-1} W,
    verified (max|V^T V - I| <= 1e-11; a Newton-Schulz step above 1e-12,
    forced here once with RLRA_SVD_VSOLVE_NS=1).  At l = 130 (3 row chunks)
    a visit is one CTA and the rotations are the V-accumulating run's, so
    sigma is bit-identical to RLRA_SVD_VSOLVE=0; at l = 300 every visit is
    split into two row-half tasks whose partial Grams are summed (another
    rounding of the same Gram: sigma within 1e-13, and bit-identical run to
    run).  U, sigma, V match the oracle with the reference's Omega (the
    exact-rank input's R-hat has a trailing block at rounding level and is
    still accepted).  A rejected solve (RLRA_SVD_VSOLVE_TOL=-1) re-runs the
    sweeps with V accumulated: U, sigma, V bit-identical to
    RLRA_SVD_VSOLVE=0."""
    import os
    import subprocess
    import sys

    from helpers import make_test_matrix, reconstruct

    m, n, p, q = 700, 500, 10, 2
    halves = k + p >= 256
    a = (make_test_matrix(m, n, np.exp(-np.arange(n) / 40.0), seed=11) if kind == "graded"
         else exact_rank(m, n, 60, seed=12))
    np.save(tmp_path / "a.npy", a)
    outs, logs = {}, {}
    for mode, extra in (("solve", {}), ("solve2", {}), ("acc", {"RLRA_SVD_VSOLVE": "0"}),
                        ("reject", {"RLRA_SVD_VSOLVE_TOL": "-1"}), ("ns", {"RLRA_SVD_VSOLVE_NS": "1"})):
        code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_1502_05366_b200 as R; "
                "a = np.load(%r); u, s, v = R.Engine(0).rsvd_v2(a, %d, %d, %d, 1, rng=R.Rng(12345)); "
                "np.savez(%r, u=u, s=s, v=v)" % (ROOT, str(tmp_path / "a.npy"), k, p, q,
                                                 str(tmp_path / ("o_%s.npz" % mode))))
        env = {**os.environ, "RLRA_SVD_KERNEL": "sgram", "RLRA_JACOBI_STATS": "1", **extra}
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert out.returncode == 0, out.stderr
        outs[mode], logs[mode] = np.load(tmp_path / ("o_%s.npz" % mode)), out.stderr
    assert "(W only)" in logs["solve"] and "accepted" in logs["solve"], logs["solve"]
    assert ("(row halves)" in logs["solve"]) == halves, logs["solve"]
    assert "(W only)" not in logs["acc"], logs["acc"]
    assert "rejected" in logs["reject"], logs["reject"]
    for key in ("u", "s", "v"):
        assert np.array_equal(outs["reject"][key], outs["acc"][key]), key
        assert np.array_equal(outs["solve"][key], outs["solve2"][key]), key  # deterministic
    uo, so, vo = orc.rsvd(a, k, p, q, 1, orc.rng(12345), 0)
    eo = np.linalg.norm(a - reconstruct(uo, so, vo))
    nz = so > 1e-12 * so[0]
    for mode in ("solve", "ns"):
        u, s, v = outs[mode]["u"], outs[mode]["s"], outs[mode]["v"]
        if halves:
            sa = outs["acc"]["s"]
            big = sa > 1e-12 * sa[0]
            assert np.max(np.abs(s[big] - sa[big]) / sa[big]) <= 1e-13, mode
        else:
            assert np.array_equal(s, outs["acc"]["s"]), mode
        assert np.max(np.abs(s[nz] - so[nz]) / so[nz]) <= 1e-10
        assert np.all(s[~nz] <= 1e-12 * so[0])
        e = np.linalg.norm(a - reconstruct(u, s, v))
        assert e <= 1.01 * eo + 1e-13 * np.linalg.norm(a), mode
        assert orthonormality_defect(u) <= 1e-11 and orthonormality_defect(v) <= 1e-11, mode
