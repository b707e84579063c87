"""The row-sharded path on the GPU engine with a real NCCL process group
(world size 1 on the single-GPU test box: the collectives run, the sums are
trivially complete).  World sizes 2-4 of the same C++ drivers run in
tests/test_gpu_dist_ranks.py (ranks on one GPU, host-staged collectives)."""
import os
import socket

import numpy as np
import pytest

import paper_1502_05366_b200 as R

pytestmark = pytest.mark.gpu


def test_native_rowsharded_rsvd_world1_matches_engine():
    """The C++ row-sharded driver (csrc/dist.cu) with a real 1-rank NCCL
    communicator: every collective runs through NCCL; the result matches the
    single-GPU engine (same Philox Omega)."""
    import torch

    from paper_1502_05366_b200 import dist as D
    from paper_1502_05366_b200.testmat import gen_test_matrix_device

    eng = R.Engine(0)
    torch.cuda.set_device(0)
    m, n, k, p, q = 6000, 3000, 100, 10, 2
    A, st = gen_test_matrix_device(eng, m, n, np.exp(-np.arange(1500) / 30.0), seed=9)
    comm = D.NcclComm(eng)
    try:
        U, S, V = D.rsvd_v2_native(comm, D.DM(A, m, n), m, k, p, q, 1, R.Omega.philox(4242))
    finally:
        comm.close()
    Ue = torch.empty(m * k, dtype=torch.float64, device="cuda")
    Ve = torch.empty(n * k, dtype=torch.float64, device="cuda")
    Se = torch.empty(k, dtype=torch.float64, device="cuda")
    eng.device_rsvd(R.RSVD_V2, A.data_ptr(), m, n, m, k, p, q, 1, R.Omega.philox(4242), Ue.data_ptr(),
                    Se.data_ptr(), Ve.data_ptr())
    s_d, s_e = S.t.cpu().numpy(), Se.cpu().numpy()
    assert np.max(np.abs(s_d - s_e) / s_e) <= 1e-10
    stn = st.cpu().numpy()
    assert np.max(np.abs(s_d[:20] - stn[:20]) / stn[:20]) <= 1e-10
    rel = eng.device_rel_error(A.data_ptr(), m, n, U.ptr, S.ptr, V.ptr, k)
    rel_e = eng.device_rel_error(A.data_ptr(), m, n, Ue.data_ptr(), Se.data_ptr(), Ve.data_ptr(), k)
    assert rel <= 1.01 * rel_e


def test_native_rowsharded_rsvd_host_shard_matches_device_shard():
    """rlra_rsvd_rowsharded with the shard in HOST memory (row-chunked upload
    under the local sketch) gives the device-shard result: same sigma, same
    reconstruction, U and V equal to rounding."""
    import torch

    from paper_1502_05366_b200 import dist as D
    from paper_1502_05366_b200.testmat import gen_test_matrix_device

    eng = R.Engine(0)
    torch.cuda.set_device(0)
    m, n, k, p, q = 5000, 2400, 80, 10, 2
    A, _ = gen_test_matrix_device(eng, m, n, np.exp(-np.arange(1200) / 25.0), seed=19)
    a_host = np.asfortranarray(A.view(n, m).t().cpu().numpy())
    comm = D.NcclComm(eng)
    try:
        U, S, V = D.rsvd_v2_native(comm, D.DM(A, m, n), m, k, p, q, 1, R.Omega.philox(77))
        uh = np.zeros((m, k), order="F")
        vh = np.zeros((n, k), order="F")
        sh = np.zeros(k)
        eng.host_rsvd_rowsharded_ptr(comm.handle, a_host.ctypes.data, m, n, m, m, k, p, q, 1, R.Omega.philox(77),
                                     uh.ctypes.data, m, sh.ctypes.data, vh.ctypes.data, n)
    finally:
        comm.close()
    s_d = S.t.cpu().numpy()
    assert np.max(np.abs(sh - s_d) / s_d) <= 1e-12
    u_d = U.t[: m * k].view(k, m).t().cpu().numpy()
    v_d = V.t[: n * k].view(k, n).t().cpu().numpy()
    assert np.linalg.norm((uh * sh) @ vh.T - (u_d * s_d) @ v_d.T) <= 1e-10 * np.linalg.norm(a_host)


def test_native_rowsharded_row_permutation_invariance():
    """The sharded driver's sums are row-order independent: permuting A's
    rows (what a different row partition does to the association order)
    leaves sigma unchanged to rounding."""
    import torch

    from paper_1502_05366_b200 import dist as D
    from paper_1502_05366_b200.testmat import gen_test_matrix_device

    eng = R.Engine(0)
    m, n, k, p, q = 4096, 2000, 64, 8, 1
    A, _ = gen_test_matrix_device(eng, m, n, np.exp(-np.arange(1000) / 20.0), seed=3)
    perm = torch.randperm(m, generator=torch.Generator().manual_seed(0)).cuda()
    Ap = A.view(n, m)[:, perm].contiguous().view(-1)
    comm = D.NcclComm(eng)
    try:
        _, S1, _ = D.rsvd_v2_native(comm, D.DM(A, m, n), m, k, p, q, 1, R.Omega.philox(5))
        _, S2, _ = D.rsvd_v2_native(comm, D.DM(Ap, m, n), m, k, p, q, 1, R.Omega.philox(5))
    finally:
        comm.close()
    s1, s2 = S1.t.cpu().numpy(), S2.t.cpu().numpy()
    assert np.max(np.abs(s1 - s2) / s1) <= 1e-10


def _world1_comm(eng):
    from paper_1502_05366_b200 import dist as D

    return D.NcclComm(eng)


@pytest.mark.parametrize("m,n,k,p", [(1500, 900, 60, 10), (3000, 1200, 120, 10)])
def test_native_rowsharded_id_cur_world1_match_engine_and_oracle(orc, m, n, k, p):
    """The row-sharded ID/CUR driver (csrc/dist.cu) on a 1-rank NCCL
    communicator: the distributed column-pivoted QR of C^T (allgathered pivot
    statistics, allreduced pivot column, positions tracked instead of column
    swaps) picks the reference's skeleton rows; jc/jr identical to the oracle
    with the reference's Omega injected."""
    from helpers import make_test_matrix, rel_fro

    eng = R.Engine(0)
    a = make_test_matrix(m, n, 10.0 ** (-8.0 * np.arange(min(m, n) // 2) / (min(m, n) // 2)), seed=11)
    comm = _world1_comm(eng)
    try:
        idg = eng.id_rand_rowsharded(comm.handle, a, 0, m, k, p, 2, 1, rng=R.Rng(12345))
        cg = eng.cur_rand_rowsharded(comm.handle, a, 0, m, k, p, 2, 1, rng=R.Rng(12345))
    finally:
        comm.close()
    ido = orc.id_rand(a, k, p, 2, 1, orc.rng(12345))
    co = orc.cur_rand(a, k, p, 2, 1, orc.rng(12345))
    np.testing.assert_array_equal(idg["jc"][:k], ido["jc"][:k])
    assert rel_fro(idg["v"], ido["v"]) <= 1e-8
    np.testing.assert_array_equal(cg["jc"][:k], co["jc"][:k])
    np.testing.assert_array_equal(cg["jr"], co["jr"][:k])
    assert abs(cg["residual"] - co["residual"]) <= 1e-6 * co["residual"] + 1e-12
    np.testing.assert_array_equal(cg["c"], a[:, cg["jc"][:k]])
    np.testing.assert_array_equal(cg["r"], a[cg["jr"], :])
    assert rel_fro(cg["u"], co["u"]) <= 1e-6
    # W: skeleton rows are exactly the identity
    np.testing.assert_array_equal(cg["w"][cg["jr"], :], np.eye(k))


def test_native_rowsharded_qb_world1_matches_engine_and_oracle(orc):
    """Row-sharded qb_blocked (csrc/dist.cu) on a 1-rank NCCL communicator:
    same adaptive rank, residual history and QB as the single-GPU engine and
    the oracle with the reference's per-block Omega substreams."""
    from helpers import make_test_matrix, rel_fro

    eng = R.Engine(0)
    m, n, b, M, tol = 700, 500, 16, 20, 1e-6
    a = make_test_matrix(m, n, (np.arange(min(m, n)) + 1.0) ** -2, seed=4)
    comm = _world1_comm(eng)
    try:
        got = eng.qb_blocked_rowsharded(comm.handle, a, m, b, M, tol, 1, 1, rng=R.Rng(12345))
    finally:
        comm.close()
    single = eng.qb_blocked(a, b, M, tol, 1, 1, rng=R.Rng(12345))
    want = orc.qb_blocked(a, b, M, tol, 1, 1, orc.rng(12345))
    assert got["ell"] == single["ell"] == want["ell"]
    assert got["tolerance_reached"] == want["reached"]
    assert abs(got["final_residual"] - want["final"]) <= 1e-6 * want["final"] + 1e-13
    np.testing.assert_allclose(got["history"], want["history"], rtol=1e-6, atol=1e-13)
    assert rel_fro(got["q"] @ got["b"], a) <= 2.0 * rel_fro(want["q"] @ want["b"], a) + 1e-14
    assert np.linalg.norm(got["q"].T @ got["q"] - np.eye(got["ell"])) <= 1e-12


@pytest.mark.parametrize("nrb", [2, 4])
def test_native_hierarchical_qb_world1_matches_single_gpu(nrb):
    """qb_hierarchical over the ranks (csrc/dist.cu) on a 1-rank NCCL
    communicator: the rank holds every slab, merges its subtree locally and
    goes through the allgather path; Q, B equal the single-GPU driver (same
    reference substreams)."""
    from helpers import make_test_matrix, rel_fro

    eng = R.Engine(0)
    m, n, b, M = 400, 150, 8, 3
    a = make_test_matrix(m, n, np.exp(-np.arange(150) / 8.0), seed=22)
    comm = _world1_comm(eng)
    try:
        got = eng.qb_hierarchical_rowsharded(comm.handle, a, m, nrb, b, M, 1, R.Rng(31))
    finally:
        comm.close()
    want = eng.qb_hierarchical(a, nrb, b, M, 1, R.Rng(31))
    assert rel_fro(got["q"], want["q"]) <= 1e-12 and rel_fro(got["b"], want["b"]) <= 1e-12
    assert abs(got["final_residual"] - want["final_residual"]) <= 1e-10 * want["final_residual"]
