"""The C++ row-sharded drivers (csrc/dist.cu) at world sizes 2, 3 and 4 on ONE
GPU.

Ranks run as threads of this process, one Engine (rlra_ctx) each, joined by an
rlra_local_group: the drivers' collectives are host-staged (each exchanged
buffer goes to pinned host memory after the rank's stream drains, is summed
in rank order, and comes back), and a GPU token keeps one rank's kernels on
the device at a time, so no kernel ever waits on another rank's kernel
(B200_PROFILING.md: such waits are not guaranteed to make progress on one
GPU).  The same orchestration code runs with NCCL in production; only the
transport of the small exchanged buffers differs.  The last test runs two
PROCESSES on the GPU with the collectives over a torch.distributed gloo
group (dist.HostComm, Python callbacks, a file-lock GPU token).

Each sharded result is checked against the single-GPU engine and the oracle
with the reference's Omega injected (every rank draws the same Omega from its
own RngState(12345)): sigma within 1e-10, residual within 1.01x, pivots
identical, replicated outputs bit-identical across ranks.
"""
import os
import socket
import threading

import numpy as np
import pytest

import paper_1502_05366_b200 as R
from helpers import make_test_matrix, rel_fro

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def run_ranks(bounds, fn, timeout=600):
    """fn(rank, eng, comm, r0, r1) on len(bounds)-1 rank threads; returns the
    per-rank results (re-raising the first rank error)."""
    world = len(bounds) - 1
    grp = R.LocalGroup(world, timeout_s=300)
    out, err = [None] * world, [None] * world

    def body(r):
        eng = R.Engine(0)
        comm = None
        try:
            comm = eng.comm_create_host(world, r, grp.collectives(r))
            out[r] = fn(r, eng, comm, int(bounds[r]), int(bounds[r + 1]))
        except BaseException as e:  # noqa: BLE001 - reported below
            err[r] = e
        finally:
            if comm is not None:
                eng.comm_destroy(comm)
            eng.close()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    assert not any(t.is_alive() for t in th), "rank threads hung"
    grp.close()
    for e in err:
        if e is not None:
            raise e
    return out


def sigma_ok(s, so):
    rel = np.abs(s - so) / so
    floor = 2.2e-16 * so[0] / so > 1e-11
    return bool(np.all((rel <= 1e-10) | (floor & (np.abs(s - so) <= 1e-13 * so[0]))))


BOUNDS = {2: [0, 1400, 3000], 3: [0, 1000, 1001, 3000], 4: [0, 700, 1500, 2300, 3000]}


@pytest.mark.parametrize("world", [2, 3, 4])
def test_rsvd_rowsharded_ranks_match_engine_and_oracle(eng, orc, world):
    m, n, k, p, q = 3000, 1200, 60, 10, 2
    a = make_test_matrix(m, n, np.exp(-np.arange(600) / 15.0), seed=41)
    b = BOUNDS[world]
    res = run_ranks(b, lambda r, e, c, r0, r1: e.rsvd_rowsharded(c, a[r0:r1], m, k, p, q, 1, rng=R.Rng(12345)))
    U = np.vstack([x[0] for x in res])
    s, V = res[0][1], res[0][2]
    for x in res[1:]:  # replicated outputs: the same bits on every rank
        assert np.array_equal(x[1], s) and np.array_equal(x[2], V)
    us, ss, vs = eng.rsvd_v2(a, k, p, q, 1, rng=R.Rng(12345))
    uo, so, vo = orc.rsvd(a, k, p, q, 1, orc.rng(12345), 0)
    assert sigma_ok(s, so) and sigma_ok(ss, so)
    e = np.linalg.norm(a - (U * s) @ V.T)
    eo = np.linalg.norm(a - (uo * so) @ vo.T)
    assert e <= 1.01 * eo, (e, eo)
    assert np.linalg.norm(U.T @ U - np.eye(k)) <= 1e-12


def test_rsvd_rowsharded_empty_host_shard(orc):
    """A rank holding no rows (host shard of 0 x n) still joins every
    collective and consumes its Omega draw: the factorization equals the
    oracle's, and every rank's RngState advanced like the reference's."""
    m, n, k, p, q = 1500, 600, 40, 10, 2
    a = make_test_matrix(m, n, np.exp(-np.arange(300) / 10.0), seed=46)
    b = [0, 0, 700, 1500]
    rngs = [R.Rng(12345) for _ in range(3)]
    res = run_ranks(b, lambda r, e, c, r0, r1: e.rsvd_rowsharded(c, a[r0:r1], m, k, p, q, 1, rng=rngs[r]))
    U = np.vstack([x[0] for x in res])
    s, V = res[0][1], res[0][2]
    uo, so, vo = orc.rsvd(a, k, p, q, 1, orc.rng(12345), 0)
    assert sigma_ok(s, so)
    assert np.linalg.norm(a - (U * s) @ V.T) <= 1.01 * np.linalg.norm(a - (uo * so) @ vo.T)
    after = [r.next_u64() for r in rngs]
    assert len(set(after)) == 1


@pytest.mark.parametrize("world", [2, 3])
def test_id_cur_rand_rowsharded_ranks_pivots_match_oracle(orc, world):
    """The distributed CPQR of C^T (allgathered pivot statistics, positions
    tracked across ranks) picks the reference's skeleton rows for any row
    partition, including a 1-row rank."""
    m, n, k, p = 3000, 1200, 80, 10
    a = make_test_matrix(m, n, 10.0 ** (-8.0 * np.arange(600) / 600), seed=43)
    b = BOUNDS[world]
    res = run_ranks(b, lambda r, e, c, r0, r1: (
        e.id_rand_rowsharded(c, a[r0:r1], r0, m, k, p, 2, 1, rng=R.Rng(12345)),
        e.cur_rand_rowsharded(c, a[r0:r1], r0, m, k, p, 2, 1, rng=R.Rng(12345))))
    ido = orc.id_rand(a, k, p, 2, 1, orc.rng(12345))
    co = orc.cur_rand(a, k, p, 2, 1, orc.rng(12345))
    for idg, cg in res:
        np.testing.assert_array_equal(idg["jc"][:k], ido["jc"][:k])
        assert rel_fro(idg["v"], ido["v"]) <= 1e-8
        np.testing.assert_array_equal(cg["jc"][:k], co["jc"][:k])
        np.testing.assert_array_equal(cg["jr"], co["jr"][:k])
        assert abs(cg["residual"] - co["residual"]) <= 1e-6 * co["residual"] + 1e-12
        np.testing.assert_array_equal(cg["r"], a[cg["jr"], :])
    C = np.vstack([cg["c"] for _, cg in res])
    np.testing.assert_array_equal(C, a[:, co["jc"][:k]])
    W = np.vstack([cg["w"] for _, cg in res])
    np.testing.assert_array_equal(W[co["jr"][:k], :], np.eye(k))


@pytest.mark.parametrize("world", [2, 4])
def test_qb_blocked_rowsharded_ranks_match_oracle(orc, world):
    m, n, bsz, M, tol = 3000, 700, 16, 30, 1e-6
    a = make_test_matrix(m, n, (np.arange(700) + 1.0) ** -2, seed=44)
    b = BOUNDS[world]
    res = run_ranks(b, lambda r, e, c, r0, r1: e.qb_blocked_rowsharded(c, a[r0:r1], m, bsz, M, tol, 1, 1,
                                                                        rng=R.Rng(12345)))
    want = orc.qb_blocked(a, bsz, M, tol, 1, 1, orc.rng(12345))
    for g in res:
        assert g["ell"] == want["ell"] and g["tolerance_reached"] == want["reached"]
        np.testing.assert_allclose(g["history"], want["history"], rtol=1e-6, atol=1e-13)
        assert np.array_equal(g["b"], res[0]["b"])
    Q = np.vstack([g["q"] for g in res])
    assert np.linalg.norm(Q.T @ Q - np.eye(Q.shape[1])) <= 1e-12
    assert rel_fro(Q @ res[0]["b"], a) <= 2.0 * rel_fro(want["q"] @ want["b"], a) + 1e-14


@pytest.mark.parametrize("world,nrb", [(2, 2), (2, 4), (4, 4)])
def test_qb_hierarchical_rowsharded_ranks_match_single_gpu(eng, world, nrb):
    """Leaves and subtree merges local, subtree roots allgathered, upper merges
    replicated (qb.hpp:211-271): Q, B equal the single-GPU tree."""
    m, n, bsz, M = 800, 150, 8, 3
    a = make_test_matrix(m, n, np.exp(-np.arange(150) / 8.0), seed=22)
    base = m // nrb
    L = nrb // world
    b = [g * L * base for g in range(world)] + [m]
    res = run_ranks(b, lambda r, e, c, r0, r1: e.qb_hierarchical_rowsharded(c, a[r0:r1], m, nrb, bsz, M, 1,
                                                                             R.Rng(31)))
    want = eng.qb_hierarchical(a, nrb, bsz, M, 1, R.Rng(31))
    Q = np.vstack([g["q"] for g in res])
    assert rel_fro(Q, want["q"]) <= 1e-12 and rel_fro(res[0]["b"], want["b"]) <= 1e-12
    for g in res:
        assert abs(g["final_residual"] - want["final_residual"]) <= 1e-10 * want["final_residual"]


def test_rsvd_rowsharded_rank_deficient_sketch_uses_tsqr(eng):
    """Exact rank 30 < l = 50, and one rank holding fewer rows than l: CholQR2
    and shifted CholQR3 break down on the sketch, the TSQR fallback
    (allgathered R factors) returns an orthonormal basis and the exact
    factorization, like the single-GPU engine's Householder fallback and the
    reference's orth (the sharded path used to raise here)."""
    m, n, k, p, r = 900, 400, 40, 10, 30
    rs = np.random.default_rng(5)
    a = np.asfortranarray(rs.standard_normal((m, r)) @ rs.standard_normal((r, n)))
    b = [0, 20, 500, 900]
    res = run_ranks(b, lambda rk, e, c, r0, r1: e.rsvd_rowsharded(c, a[r0:r1], m, k, p, 2, 1, rng=R.Rng(12345)))
    U = np.vstack([x[0] for x in res])
    s, V = res[0][1], res[0][2]
    us, ss, vs = eng.rsvd_v2(a, k, p, 2, 1, rng=R.Rng(12345))
    assert np.max(np.abs(s[:r] - ss[:r]) / ss[:r]) <= 1e-10
    assert np.all(s[r:] <= 1e-10 * s[0])
    assert np.linalg.norm(a - (U * s) @ V.T) <= 1e-11 * np.linalg.norm(a)
    assert np.linalg.norm(U[:, :r].T @ U[:, :r] - np.eye(r)) <= 1e-12


def test_gen_test_matrix_rowsharded_ranks_equal_single_gpu(eng):
    """rlra_gen_test_matrix_rowsharded: U's Philox rows orthonormalised across
    the ranks; the assembled matrix equals the single-GPU generator's."""
    import torch

    m, n, sig = 2000, 600, np.exp(-np.arange(300) / 30.0)
    b = [0, 700, 701, 2000]

    def gen(r, e, c, r0, r1):
        A = torch.empty(max((r1 - r0) * n, 1), dtype=torch.float64, device="cuda")
        e.device_gen_test_matrix_rowsharded(c, r0, r1 - r0, m, n, sig, 7, 1e-6, A.data_ptr(), max(1, r1 - r0))
        e.synchronize()
        return A[: (r1 - r0) * n].view(n, r1 - r0).t().cpu().numpy()

    a = np.vstack(run_ranks(b, gen))
    A1 = torch.empty(m * n, dtype=torch.float64, device="cuda")
    eng.device_gen_test_matrix(m, n, sig, 7, 1e-6, A1.data_ptr(), m)
    eng.synchronize()
    a1 = A1.view(n, m).t().cpu().numpy()
    assert np.linalg.norm(a - a1) <= 1e-13 * np.linalg.norm(a1)


def test_local_group_mismatched_collective_fails_instead_of_hanging():
    """A rank that leaves the protocol (different work on different ranks)
    surfaces as RLRA_ENCCL on every rank within the group timeout, not a hang."""
    grp = R.LocalGroup(2, timeout_s=30.0)
    errs = [None, None]

    def body(r):
        e = R.Engine(0)
        c = e.comm_create_host(2, r, grp.collectives(r))
        try:
            a = make_test_matrix(300 if r == 0 else 200, 100, np.exp(-np.arange(100) / 5.0), seed=1)
            if r == 0:
                e.rsvd_rowsharded(c, a, 500, 10, 5, 2, 1, rng=R.Rng(1))
            else:
                e.qb_blocked_rowsharded(c, a, 500, 8, 3, 0.0, 0, 1, rng=R.Rng(1))
        except R.RlraError as x:
            errs[r] = x
        finally:
            e.comm_destroy(c)
            e.close()

    th = [threading.Thread(target=body, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(120)
    assert not any(t.is_alive() for t in th)
    grp.close()
    assert all(isinstance(x, R.RlraError) for x in errs), errs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, lock, out):
    import sys

    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    import torch.distributed as dist

    import paper_1502_05366_b200 as RR
    from helpers import make_test_matrix as mk
    from paper_1502_05366_b200 import dist as D

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        e = RR.Engine(0)
        comm = D.HostComm(e, share_gpu=True, lock_path=lock)
        m, n, k, p, q = 2000, 800, 40, 10, 2
        a = mk(m, n, np.exp(-np.arange(400) / 12.0), seed=45)
        r0, r1 = [0, 900, 2000][rank], [0, 900, 2000][rank + 1]
        u, s, v = e.rsvd_rowsharded(comm.handle, a[r0:r1], m, k, p, q, 1, rng=RR.Rng(12345))
        np.savez(os.path.join(out, f"g{rank}.npz"), u=u, s=s, v=v)
        comm.close()
    finally:
        dist.destroy_process_group()


def test_rsvd_rowsharded_two_processes_over_gloo(tmp_path, eng, orc):
    """Two processes on the GPU, the C++ driver's collectives over a gloo
    process group through Python callbacks (dist.HostComm)."""
    import torch.multiprocessing as mp

    port = _free_port()
    mp.spawn(_gloo_worker, args=(2, port, str(tmp_path / "tok.lock"), str(tmp_path)), nprocs=2, join=True)
    parts = [np.load(os.path.join(tmp_path, f"g{r}.npz")) for r in range(2)]
    m, n, k, p, q = 2000, 800, 40, 10, 2
    a = make_test_matrix(m, n, np.exp(-np.arange(400) / 12.0), seed=45)
    assert np.array_equal(parts[0]["s"], parts[1]["s"]) and np.array_equal(parts[0]["v"], parts[1]["v"])
    U = np.vstack([x["u"] for x in parts])
    s, V = parts[0]["s"], parts[0]["v"]
    uo, so, vo = orc.rsvd(a, k, p, q, 1, orc.rng(12345), 0)
    assert sigma_ok(s, so)
    assert np.linalg.norm(a - (U * s) @ V.T) <= 1.01 * np.linalg.norm(a - (uo * so) @ vo.T)
