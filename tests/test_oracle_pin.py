"""Pins for the CPU oracle (CPU-only; no GPU needed).

1. The C restatement (oracle/rlra_oracle.c) reproduces the golden vectors
   that tests/golden/make_golden.py produced with the unmodified reference,
   bit for bit.
2. Where oracle/_ref (the reference headers compiled by oracle/Makefile) is
   present, the restatement matches it bit for bit on fresh random inputs
   for every entry point.
3. The reference's own known-answer tests hold on the oracle.
"""
import os

import numpy as np
import pytest

import _oracle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")


@pytest.fixture(scope="module")
def g():
    return np.load(GOLD)


def same(x, y):
    return np.array_equal(np.asarray(x), np.asarray(y))


def test_golden_rng_stream(orc, g):
    r = orc.rng(12345)
    assert same(orc.gaussian(7, 3, r), g["rng_12345_7x3"])
    assert same(orc.gaussian(5, 1, r), g["rng_12345_next_5x1"])
    r = orc.rng(42)
    c1, c2 = orc.substream(r), orc.substream(r)
    assert same(orc.gaussian(4, 2, c1), g["rng_42_sub1_4x2"])
    assert same(orc.gaussian(4, 2, c2), g["rng_42_sub2_4x2"])


def test_golden_matmul(orc, g):
    assert same(orc.matmul(g["mm_a"], g["mm_b"]), g["mm_nn"])
    assert same(orc.matmul(g["mm_a"], g["mm_tn_b"], True, False), g["mm_tn"])
    assert same(orc.matmul(g["mm_a"], g["mm_nt_b"], False, True), g["mm_nt"])


def test_golden_qr_family(orc, g):
    q, _, _ = orc.compact_qr(np.array([[3.0], [4.0]]))
    assert same(q, g["orth_34"])
    assert abs(q[0, 0] - 0.6) <= 1e-15 and abs(q[1, 0] - 0.8) <= 1e-15
    q, r, _ = orc.compact_qr(g["qr_in"])
    assert same(q, g["qr_q"]) and same(r, g["qr_r"])
    f = orc.pivoted_qr(np.diag([3.0, 2.0, 1.0]), 2)
    assert same(f["perm"], g["cpqr_diag_perm"]) and list(f["perm"][:2]) == [0, 1]
    assert f["residual"] == g["cpqr_diag_res"][0] and abs(f["residual"] - 1.0) <= 1e-14
    f = orc.pivoted_qr(g["cpqr_in"], 8)
    assert same(f["perm"], g["cpqr_perm"]) and same(f["s1"], g["cpqr_s1"])
    assert f["residual"] == g["cpqr_res"][0]
    t, cl = orc.upper_tri_solve(np.array([[1e8, 0.0], [0.0, 1e-8]]), np.array([[1.0], [1.0]]))
    assert cl and same(t, g["trisolve_clamp"]) and t[1, 0] == 1e4


def test_golden_jacobi(orc, g):
    _, s, _ = orc.small_svd(np.diag([2.0, -3.0]))
    assert same(s, g["svd_diag_sigma"]) and list(s) == [3.0, 2.0]
    u, s, v = orc.small_svd(g["svd_in"])
    assert same(u, g["svd_u"]) and same(s, g["svd_s"]) and same(v, g["svd_v"])


def test_golden_algorithms(orc, g):
    A = g["A"]
    for var, name in [(0, "v2"), (1, "v1"), (2, "basic")]:
        u, s, v = orc.rsvd(A, 8, 4, 2, 1, orc.rng(12345), var)
        assert same(u, g[f"rsvd_{name}_u"]) and same(s, g[f"rsvd_{name}_s"])
        assert same(v, g[f"rsvd_{name}_v"])
    f = orc.qb_blocked(A, 5, 6, 1e-3, 1, 1, orc.rng(12345))
    assert f["ell"] == g["qb_ell"][0]
    assert same(f["q"], g["qb_q"]) and same(f["b"], g["qb_b"]) and same(f["history"], g["qb_hist"])
    _, s, _ = orc.svd_from_qb(f["q"], f["b"], 0, 0)
    assert same(s, g["svdqb_s"])
    f = orc.id_rand(A, 10, 5, 2, 1, orc.rng(12345))
    assert same(f["jc"], g["idrand_jc"]) and same(f["v"], g["idrand_v"])
    assert f["qr_residual"] == g["idrand_res"][0]
    f = orc.cur_rand(A, 10, 5, 2, 1, orc.rng(12345))
    for key in ("jc", "jr", "c", "u", "r"):
        assert same(f[key], g[f"cur_{key}"]), key
    assert f["residual"] == g["cur_res"][0] and f["qr_residual"] == g["cur_res"][1]


@pytest.mark.skipif(not _oracle.have_ref(), reason="oracle/_ref not built (no /root/reference)")
def test_restatement_matches_reference_bitwise(orc):
    ref = _oracle.ref()
    rs = np.random.default_rng(0)
    A = np.asfortranarray(rs.standard_normal((45, 33)))
    for ta in (0, 1):
        for tb in (0, 1):
            B = rs.standard_normal(((33 if not ta else 45), 7) if not tb else (7, (33 if not ta else 45)))
            assert same(orc.matmul(A, B, ta, tb), ref.matmul(A, B, ta, tb))
    for x, y in zip(orc.compact_qr(A), ref.compact_qr(A)):
        assert same(x, y)
    for k, tol in [(12, 0.0), (0, 0.5)]:
        po, pr = orc.pivoted_qr(A, k, tol), ref.pivoted_qr(A, k, tol)
        assert all(same(po[key], pr[key]) for key in po)
    for M in (A, A.T):
        for x, y in zip(orc.small_svd(M), ref.small_svd(M)):
            assert same(x, y)
    S = A.T @ A
    for x, y in zip(orc.sym_eig(S), ref.sym_eig(S)):
        assert same(x, y)
    for left in (False, True):
        ro, rr = orc.rng(5), ref.rng(5)
        assert same(orc.sample(A, 9, 2, 2, ro, left), ref.sample(A, 9, 2, 2, rr, left))
    for var in (0, 1, 2):
        for x, y in zip(orc.rsvd(A, 7, 3, 1, 1, orc.rng(7), var), ref.rsvd(A, 7, 3, 1, 1, ref.rng(7), var)):
            assert same(x, y)
    qo = orc.qb_blocked(A, 4, 8, 1e-2, 1, 2, orc.rng(9), True)
    qr_ = ref.qb_blocked(A, 4, 8, 1e-2, 1, 2, ref.rng(9), True)
    assert all(same(qo[key], qr_[key]) for key in qo)
    for vnum in (0, 1):
        for x, y in zip(orc.svd_from_qb(qo["q"], qo["b"], 0, vnum), ref.svd_from_qb(qr_["q"], qr_["b"], 0, vnum)):
            assert same(x, y)
    io, ir = orc.id_column(A, 10), ref.id_column(A, 10)
    assert all(same(io[key], ir[key]) for key in io)
    io, ir = orc.id_rand(A, 10, 5, 2, 1, orc.rng(11)), ref.id_rand(A, 10, 5, 2, 1, ref.rng(11))
    assert all(same(io[key], ir[key]) for key in io)
    co, cr = orc.cur_rand(A, 8, 4, 1, 1, orc.rng(13)), ref.cur_rand(A, 8, 4, 1, 1, ref.rng(13))
    assert all(same(co[key], cr[key]) for key in co)


def test_oracle_reference_kats(orc):
    """Reference known answers on the oracle (tests/test_qr.cpp, test_jacobi.cpp)."""
    rs = np.random.default_rng(26)
    a = rs.standard_normal((20, 2)) @ rs.standard_normal((20, 2)).T
    f = orc.pivoted_qr(a, 0, 1e-10)
    assert f["frank"] == 2 and f["reached"]
    c = rs.standard_normal((6, 1))
    _, r, deg = orc.compact_qr(np.hstack([c, np.zeros((6, 1))]))
    assert deg and r[1, 1] == 0.0
    with pytest.raises(_oracle.OracleError):
        orc.upper_tri_solve(np.array([[1.0, 2.0], [0.0, 0.0]]), np.ones((2, 1)))
    a = np.diag([1.0, 1e-15])
    with pytest.raises(_oracle.OracleError) as e:
        orc.rsvd(a, 2, 0, 0, 1, orc.rng(23), 1)
    assert "use v2" in e.value.msg
    _, s, _ = orc.rsvd(a, 2, 0, 0, 1, orc.rng(23), 0)
    assert abs(s[1] - 1e-15) <= 1e-21
