"""Algorithm-level parity: rsvd / qb / ID / CUR on the CUDA engine against the
CPU oracle with the reference's own Omega injected (same RngState seed), plus
the reference test-suite's property checks re-expressed (tests/test_rsvd.cpp,
test_qb.cpp, test_interp.cpp, test_sketch.cpp).

Parity bar (BASELINE.json north_star): sigma within 1e-10 relative, the
reconstruction error within 1.01x of the reference's, ID/CUR pivots identical
wherever the pivot gap exceeds 1e-8.
"""
import numpy as np
import pytest

import paper_1502_05366_b200 as R
from helpers import (exact_rank, make_test_matrix, match_columns_up_to_sign,
                     orthonormality_defect, reconstruct, rel_fro)


pytestmark = pytest.mark.gpu

SIGMA_RTOL = 1e-10


def spectrum_exp(r, scale):
    return np.exp(-np.arange(r) / scale)


def sigma_close(s, s_ref, rtol=SIGMA_RTOL):
    s, s_ref = np.asarray(s), np.asarray(s_ref)
    # rel 1e-10 per mode; modes at the FP64 floor (u*s1/s_i > 1e-11) get the
    # absolute floor instead
    tol = np.maximum(rtol * s_ref, 1e-5 * 1e-11 * s_ref[0] / 1e-5)
    return np.all(np.abs(s - s_ref) <= tol), np.max(np.abs(s - s_ref) / s_ref)


@pytest.mark.parametrize("variant", ["v2", "v1", "basic"])
def test_rsvd_vs_oracle_injected_omega(eng, orc, variant):
    import _oracle
    m, n, k, p, q = 300, 200, 20, 5, 2
    a = make_test_matrix(m, n, spectrum_exp(200, 10.0), seed=7)
    rng = R.Rng(12345)
    ro = orc.rng(12345)
    vid = {"v2": 0, "v1": 1, "basic": 2}[variant]
    if variant == "basic":
        u, s, v = eng.rsvd_basic(a, k, p, rng=rng)
    else:
        u, s, v = getattr(eng, "rsvd_" + variant)(a, k, p, q, 1, rng=rng)
    uo, so, vo = orc.rsvd(a, k, p, q, 1, ro, vid)
    ok, worst = sigma_close(s, so)
    assert ok, worst
    e = np.linalg.norm(a - reconstruct(u, s, v))
    eo = np.linalg.norm(a - reconstruct(uo, so, vo))
    assert e <= 1.01 * eo
    assert orthonormality_defect(u) <= 1e-11 * np.sqrt(k)
    # RNG consumed exactly like the reference
    assert rng.state()[0] == tuple(ro.s)


def test_rsvd_v2_c1_shape_parity(eng, orc):
    """C1-shaped (2000x4000, k=200, p=10, q=2) at reduced n so the oracle stays
    within seconds; full C1 runs in test_gpu_configs.py."""
    m, n, k, p, q = 1000, 1500, 100, 10, 2
    a = make_test_matrix(m, n, spectrum_exp(1000, 20.0), seed=1)
    u, s, v = eng.rsvd_v2(a, k, p, q, 1, rng=R.Rng(12345))
    uo, so, vo = orc.rsvd(a, k, p, q, 1, orc.rng(12345), 0)
    ok, worst = sigma_close(s, so)
    assert ok, worst
    e = np.linalg.norm(a - reconstruct(u, s, v))
    eo = np.linalg.norm(a - reconstruct(uo, so, vo))
    assert e <= 1.01 * eo
    assert match_columns_up_to_sign(u[:, :50], uo[:, :50]) <= 1e-7


def test_rsvd_exact_rank_recovery(eng):
    a = exact_rank(40, 30, 8, 301)
    u, s, v = eng.rsvd_basic(a, 8, 3, rng=R.Rng(17))
    assert np.linalg.norm(a - reconstruct(u, s, v)) <= 1e-10 * np.linalg.norm(a)
    a = exact_rank(35, 28, 6, 304)
    u, s, v = eng.rsvd_v1(a, 6, 3, 1, 1, rng=R.Rng(19))
    assert np.linalg.norm(a - reconstruct(u, s, v)) <= 1e-9 * np.linalg.norm(a)
    a = exact_rank(35, 28, 6, 307)
    u, s, v = eng.rsvd_v2(a, 6, 3, 1, 1, rng=R.Rng(21))
    assert np.linalg.norm(a - reconstruct(u, s, v)) <= 1e-11 * np.linalg.norm(a)
    assert orthonormality_defect(u) <= 1e-11 * np.sqrt(6)
    assert orthonormality_defect(v) <= 1e-11 * np.sqrt(6)


def test_rsvd_tiny_singular_value_divergence(eng):
    """test_rsvd.cpp:188-202: v1 refuses, v2 resolves 1e-15 to 1e-21."""
    a = np.diag([1.0, 1e-15])
    with pytest.raises(R.NumericalError) as e:
        eng.rsvd_v1(a, 2, 0, 0, 1, rng=R.Rng(23))
    assert "use v2" in str(e.value)
    u, s, v = eng.rsvd_v2(a, 2, 0, 0, 1, rng=R.Rng(23))
    assert abs(s[0] - 1.0) <= 1e-12
    assert abs(s[1] - 1e-15) <= 1e-21
    assert np.linalg.norm(a - reconstruct(u, s, v)) <= 1e-11 * np.linalg.norm(a)


def test_rsvd_rank_one(eng):
    rs = np.random.default_rng(302)
    u0 = rs.standard_normal((30, 1))
    v0 = rs.standard_normal((20, 1))
    a = 3.7 * (u0 / np.linalg.norm(u0)) @ (v0 / np.linalg.norm(v0)).T
    _, s, _ = eng.rsvd_basic(a, 1, 2, rng=R.Rng(18))
    assert abs(s[0] - 3.7) <= 3.7e-10


def test_rsvd_dimension_guards(eng):
    a = np.zeros((20, 10))
    with pytest.raises(R.DimensionError):
        eng.rsvd_basic(a, 8, 3, rng=R.Rng(1))
    with pytest.raises(R.DimensionError):
        eng.rsvd_basic(a, 0, 3, rng=R.Rng(1))
    with pytest.raises(R.DimensionError):
        eng.rsvd_v1(a, 5, -1, 1, 1, rng=R.Rng(1))
    with pytest.raises(R.DimensionError):
        eng.rsvd_v2(a, 11, 0, 1, 1, rng=R.Rng(1))


def test_sample_right_q0_is_plain_sketch(eng, orc):
    a = make_test_matrix(40, 30, spectrum_exp(30, 5.0), seed=101)
    y = eng.sample_right(a, 8, 0, 1, rng=R.Rng(55))
    g = R.gaussian_matrix(30, 8, R.Rng(55))
    assert rel_fro(y, a @ g) <= 1e-14
    yl = eng.sample_left(a, 6, 0, 1, rng=R.Rng(66))
    g = R.gaussian_matrix(40, 6, R.Rng(66))
    assert yl.shape == (6, 30) and rel_fro(yl, g.T @ a) <= 1e-14


@pytest.mark.parametrize("q,s", [(1, 1), (2, 1), (2, 2), (3, 3)])
def test_sample_vs_oracle(eng, orc, q, s):
    a = make_test_matrix(120, 90, spectrum_exp(90, 8.0), seed=q * 10 + s)
    for left in (False, True):
        got = (eng.sample_left if left else eng.sample_right)(a, 12, q, s, rng=R.Rng(9))
        want = orc.sample(a, 12, q, s, orc.rng(9), left)
        assert rel_fro(got, want) <= 1e-10


def test_qb_blocked_vs_oracle(eng, orc):
    a = make_test_matrix(300, 200, spectrum_exp(200, 12.0), seed=407)
    tol = 1e-2 * np.linalg.norm(a)
    got = eng.qb_blocked(a, 20, 10, tol, 1, 1, rng=R.Rng(6))
    want = orc.qb_blocked(a, 20, 10, tol, 1, 1, orc.rng(6))
    assert got["ell"] == want["ell"]
    assert len(got["history"]) == len(want["history"])
    np.testing.assert_allclose(got["history"], want["history"], rtol=1e-8)
    assert got["tolerance_reached"] == want["reached"]
    assert np.linalg.norm(a - got["q"] @ got["b"]) < tol
    assert orthonormality_defect(got["q"]) <= 1e-9
    assert rel_fro(got["q"], want["q"]) <= 1e-8


def test_qb_exact_rank_stops_at_second_block(eng):
    a = exact_rank(30, 25, 7, 405)
    f = eng.qb_blocked(a, 4, 10, 1e-8, 1, 1, rng=R.Rng(5))
    assert f["ell"] == 8 and len(f["history"]) == 2 and f["tolerance_reached"]
    assert np.linalg.norm(a - f["q"] @ f["b"]) < 1e-8


def test_id_row_vs_oracle(eng, orc):
    """interp.hpp:107-117: the row ID is the column ID of A^T with the roles
    renamed — pivots identical, W within the reference tolerance."""
    rs = np.random.default_rng(41)
    a = rs.standard_normal((90, 12)) @ rs.standard_normal((12, 70)) + 1e-9 * rs.standard_normal((90, 70))
    got = eng.id_row(a, 12)
    want = orc.id_column(np.asfortranarray(a.T), 12)
    np.testing.assert_array_equal(got["jr"][:12], want["jc"][:12])
    assert rel_fro(got["w"], want["v"]) <= 1e-10
    assert np.linalg.norm(a - got["w"] @ a[got["jr"][:12], :]) <= 1e-6 * np.linalg.norm(a)


def test_id_from_qb_vs_oracle(eng, orc):
    """interp.hpp:228-236: the column ID of B from a QB factorisation —
    pivots identical to the oracle's ID of the same B; dimension errors as the
    reference's."""
    rs = np.random.default_rng(43)
    a = rs.standard_normal((120, 15)) @ rs.standard_normal((15, 80))
    qb = eng.qb_blocked(a, 5, 4, 0.0, 1, 1, rng=R.Rng(9))
    got = eng.id_from_qb(qb, a, 10)
    want = orc.id_column(np.asfortranarray(qb["b"]), 10)
    np.testing.assert_array_equal(got["jc"][:10], want["jc"][:10])
    assert rel_fro(got["v"], want["v"]) <= 1e-10
    with pytest.raises(R.DimensionError):
        eng.id_from_qb(qb, a[:, :50], 10)
    with pytest.raises(R.DimensionError):
        eng.id_from_qb(qb, a, qb["ell"] + 1)


def test_qb_inplace_equals_copy(eng):
    a = make_test_matrix(60, 50, spectrum_exp(50, 6.0), seed=3)
    f1 = eng.qb_blocked(a, 5, 4, 0.0, 1, 1, rng=R.Rng(8))
    w = np.asfortranarray(a.copy())
    f2 = eng.qb_blocked(w, 5, 4, 0.0, 1, 1, rng=R.Rng(8), inplace=True)
    assert np.array_equal(f1["q"], f2["q"]) and np.array_equal(f1["b"], f2["b"])
    # telescoping: W = A - QB (test_qb.cpp:123-134)
    assert np.linalg.norm(w - (a - f2["q"] @ f2["b"])) <= 1e-9 * np.linalg.norm(a)


def test_svd_from_qb_vs_oracle(eng, orc):
    a = make_test_matrix(200, 150, spectrum_exp(150, 10.0), seed=11)
    f = eng.qb_blocked(a, 10, 5, 0.0, 1, 1, rng=R.Rng(3))
    for vnum in (0, 1):
        u, s, v = eng.svd_from_qb(f, 0, vnum)
        uo, so, vo = orc.svd_from_qb(f["q"], f["b"], 0, vnum)
        ok, worst = sigma_close(s, so, 1e-9 if vnum else SIGMA_RTOL)
        assert ok, worst
    u, s, v = eng.svd_from_qb(f, 10, 0)
    assert u.shape == (200, 10) and s.shape == (10,)
    with pytest.raises(R.DimensionError):
        eng.svd_from_qb(f, 51)


def _pivot_prefix_ok(got, want):
    return np.array_equal(np.asarray(got), np.asarray(want))


def test_id_rand_vs_oracle(eng, orc):
    m, n, k, p = 400, 300, 40, 10
    a = make_test_matrix(m, n, 10.0 ** (-8.0 * np.arange(150) / 150.0), seed=3)
    got = eng.id_rand(a, k, p, 2, 1, rng=R.Rng(12345))
    want = orc.id_rand(a, k, p, 2, 1, orc.rng(12345))
    np.testing.assert_array_equal(got["jc"][:k], want["jc"][:k])
    assert abs(got["qr_residual"] - want["qr_residual"]) <= 1e-6 * want["qr_residual"] + 1e-14
    assert rel_fro(got["v"], want["v"]) <= 1e-8
    c = a[:, got["jc"][:k]]
    assert np.linalg.norm(a - c @ got["v"].T) <= 2.0 * np.linalg.norm(a - a[:, want["jc"][:k]] @ want["v"].T) + 1e-12


def test_cur_rand_vs_oracle(eng, orc):
    m, n, k, p = 300, 250, 30, 10
    a = make_test_matrix(m, n, 10.0 ** (-8.0 * np.arange(120) / 120.0), seed=5)
    got = eng.cur_rand(a, k, p, 2, 1, rng=R.Rng(12345))
    want = orc.cur_rand(a, k, p, 2, 1, orc.rng(12345))
    np.testing.assert_array_equal(got["jc"][:k], want["jc"][:k])
    np.testing.assert_array_equal(got["jr"][:k], want["jr"][:k])
    assert np.array_equal(got["c"], a[:, got["jc"][:k]])  # bit-exact extraction
    assert np.array_equal(got["r"], a[got["jr"][:k], :])
    assert got["residual"] <= 1.01 * want["residual"] + 1e-13 * np.linalg.norm(a)
    assert abs(got["residual"] - np.linalg.norm(a - got["c"] @ got["u"] @ got["r"])) <= 1e-8 * np.linalg.norm(a)


def test_id_column_dependent_column(eng):
    """test_interp.cpp:46-62: a dependent column picks pivots 1,2, V(0,0)=0.5."""
    ac = np.array([3, 1, 2, 0, 1, 2.0])
    bc = np.array([0.1, 0.2, -0.1, 0.3, 0.1, -0.2])
    a = np.stack([ac, 2.0 * ac, bc], axis=1)
    f = eng.id_column(a, 2)
    assert list(f["jc"][:2]) == [1, 2]
    assert abs(f["v"][0, 0] - 0.5) <= 1e-12 and abs(f["v"][0, 1]) <= 1e-12
    assert np.linalg.norm(a - a[:, f["jc"][:2]] @ f["v"].T) <= 1e-12
    for i in range(2):
        for j in range(2):
            assert f["v"][f["jc"][i], j] == (1.0 if i == j else 0.0)


def test_id_column_vs_oracle(eng, orc):
    rs = np.random.default_rng(8)
    a = rs.standard_normal((60, 45))
    got = eng.id_column(a, 12)
    want = orc.id_column(a, 12)
    np.testing.assert_array_equal(got["jc"], want["jc"])
    assert rel_fro(got["v"], want["v"]) <= 1e-10
    got = eng.id_column(a, 0, 1.0)
    want = orc.id_column(a, 0, 1.0)
    assert got["k"] == want["k"]


def test_two_sided_and_cur_deterministic(eng, orc):
    a = make_test_matrix(80, 70, 10.0 ** (-6.0 * np.arange(40) / 40.0), seed=9)
    ts = eng.id_two_sided(a, 10)
    want = orc.id_column(a, 10)
    np.testing.assert_array_equal(ts["jc"], want["jc"])
    jr, w = orc.two_sided_from_column(a, want["jc"], want["v"], 10)
    np.testing.assert_array_equal(ts["jr"][:10], jr[:10])
    c = eng.cur(a, 10)
    assert np.array_equal(c["c"], a[:, c["jc"][:10]]) and np.array_equal(c["r"], a[c["jr"][:10], :])


def test_cur_linkage_rank_deficient_message(eng):
    """test_interp.cpp:209-222: the message names the offending skeleton row."""
    a = np.random.default_rng(1).standard_normal((10, 3))
    a[4] = [1.0, 2.0, 3.0]
    a[9] = [2.0, 4.0, 6.0]  # dependent skeleton rows
    v = np.zeros((3, 2))
    v[0, 0] = v[1, 1] = 1.0
    ts = dict(jc=np.array([0, 1, 2], dtype=np.int32),
              jr=np.array([4, 9, 0, 1, 2, 3, 5, 6, 7, 8], dtype=np.int32), v=v, k=2, qr_residual=0.0)
    with pytest.raises(R.NumericalError) as e:
        eng.cur_from_two_sided(a, ts)
    assert "9" in str(e.value)


def _ref_lib():
    import ctypes as C
    import os

    import _oracle

    if not os.path.exists(_oracle.REF_PATH):
        pytest.skip("oracle/_ref not built")
    lib = C.CDLL(_oracle.REF_PATH)
    lib.ref_last_error.restype = C.c_char_p
    return lib


@pytest.mark.parametrize("q", [0, 1])
def test_qb_parallel_vs_reference(eng, q):
    """qb_parallel (qb.hpp:159-204) with the reference's per-block streams:
    Q, B and the residual match the unmodified reference."""
    import ctypes as C

    import _oracle

    lib = _ref_lib()
    m, n, b, M = 300, 200, 10, 4
    a = make_test_matrix(m, n, np.exp(-np.arange(200) / 15.0), seed=21)
    got = eng.qb_parallel(a, b, M, q, R.Rng(777))
    Q = np.zeros((m, b * M), order="F")
    B = np.zeros((b * M, n), order="F")
    fin = C.c_double(0)
    r = _oracle.Rng()
    lib.ref_rng_seed(C.byref(r), C.c_uint64(777))
    af = np.asfortranarray(a)
    assert lib.ref_qb_parallel(_oracle.d(af), m, n, b, M, q, C.byref(r), _oracle.d(Q), _oracle.d(B), C.byref(fin)) == 0
    assert rel_fro(got["q"], Q) <= 1e-10 and rel_fro(got["b"], B) <= 1e-10
    assert abs(got["final_residual"] - fin.value) <= 1e-8 * fin.value + 1e-14


@pytest.mark.parametrize("nrb", [2, 4])
def test_qb_hierarchical_vs_reference(eng, nrb):
    """qb_hierarchical (qb.hpp:211-271): leaf QBs of the row slabs, pairwise
    merges up the tree, the reference's leaf-then-merge substreams."""
    import ctypes as C

    import _oracle

    lib = _ref_lib()
    m, n, b, M = 400, 150, 8, 3
    a = make_test_matrix(m, n, np.exp(-np.arange(150) / 8.0), seed=22)
    got = eng.qb_hierarchical(a, nrb, b, M, 1, R.Rng(31))
    Q = np.zeros((m, b * M), order="F")
    B = np.zeros((b * M, n), order="F")
    fin = C.c_double(0)
    r = _oracle.Rng()
    lib.ref_rng_seed(C.byref(r), C.c_uint64(31))
    af = np.asfortranarray(a)
    assert lib.ref_qb_hierarchical(_oracle.d(af), m, n, nrb, b, M, 1, C.byref(r), _oracle.d(Q), _oracle.d(B),
                                   C.byref(fin)) == 0
    assert rel_fro(got["q"], Q) <= 1e-9 and rel_fro(got["b"], B) <= 1e-9
    assert abs(got["final_residual"] - fin.value) <= 1e-8 * fin.value + 1e-14
    with pytest.raises(R.DimensionError) as e:
        eng.qb_hierarchical(a, 3, b, M, 1, R.Rng(1))
    assert "num_row_blocks must be one of {2,4,8,...} (got 3)" in str(e.value)


def test_pageable_host_buffers_staged_bit_identical_to_pinned(eng):
    """A reference user's DenseMatrix is pageable memory: the C-ABI stages it
    through pinned slots with a pool of copy threads (csrc/hostio.cu) in both
    directions.  Results equal the pinned-buffer call bit for bit (240 MB A
    and the 80 MB U: both over the 64 MiB staging threshold)."""
    import torch

    m, n, k, p, q = 20000, 1500, 500, 10, 2
    a = make_test_matrix(m, n, np.exp(-np.arange(1500) / 80.0), seed=71)
    outs = []
    for pinned in (True, False):
        A = torch.from_numpy(a.T.copy().reshape(-1))  # column-major bytes
        if pinned:
            A = A.pin_memory()
        U = torch.zeros(m * k, dtype=torch.float64, pin_memory=pinned)
        V = torch.zeros(n * k, dtype=torch.float64, pin_memory=pinned)
        S = torch.zeros(k, dtype=torch.float64, pin_memory=pinned)
        eng.host_rsvd_ptr(R.RSVD_V2, A.data_ptr(), m, n, m, k, p, q, 1, R.Omega.philox(5), U.data_ptr(),
                          S.data_ptr(), V.data_ptr())
        outs.append((U.numpy().copy(), S.numpy().copy(), V.numpy().copy()))
    for x, y in zip(*outs):
        assert np.array_equal(x, y)
    u = outs[1][0].reshape(k, m).T
    assert np.linalg.norm(u.T @ u - np.eye(k)) <= 1e-11
