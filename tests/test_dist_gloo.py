"""The row-sharded multi-GPU orchestration (tests/_dist_mirror.py, the Python restatement of csrc/dist.cu) at
world size 2 over gloo on CPU, with the numpy stand-in backend: the sharded
run must reproduce the single-process run of the same algorithm (identical
Omega, different association order of the sums) and the true spectrum."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix(m, n):
    rs = np.random.default_rng(5)
    r = min(m, n)
    U, _ = np.linalg.qr(rs.standard_normal((m, r)))
    V, _ = np.linalg.qr(rs.standard_normal((n, r)))
    return np.asfortranarray((U * np.exp(-np.arange(r) / 3.0)) @ V.T)


def _worker(rank, world, port, m, n, k, p, q, out_dir):
    import sys

    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from _dist_numpy import NM, NumpyBackend, OmegaSeed

    import _dist_mirror as D

    a = _matrix(m, n)
    bounds = np.linspace(0, m, world + 1).astype(int)
    r0, r1 = bounds[rank], bounds[rank + 1]
    be = NumpyBackend()
    U, s, V = D.rsvd_v2_rowsharded(be, NM(a[r0:r1]), m, k, p, q, 1, OmegaSeed(77))
    Q = D.orth_dist(be, NM(a[r0:r1, :30]))
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), U=U.a, s=s.a[:, 0], V=V.a, r0=r0, r1=r1,
             Q=Q.a, allreduces=be.allreduces)
    dist.destroy_process_group()


def _run(world, m, n, k, p, q, tmp):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, m, n, k, p, q, str(tmp)), nprocs=world, join=True)
    parts = [np.load(os.path.join(tmp, f"r{r}.npz")) for r in range(world)]
    U = np.vstack([x["U"] for x in parts])
    Q = np.vstack([x["Q"] for x in parts])
    return U, parts[0]["s"][:k], parts[0]["V"], Q, parts


@pytest.mark.timeout(300)
def test_rowsharded_rsvd_world2_matches_world1(tmp_path):
    m, n, k, p, q = 240, 120, 12, 6, 2
    d1, d2 = tmp_path / "w1", tmp_path / "w2"
    d1.mkdir()
    d2.mkdir()
    U1, s1, V1, Q1, _ = _run(1, m, n, k, p, q, d1)
    U2, s2, V2, Q2, parts = _run(2, m, n, k, p, q, d2)
    # replicated outputs agree across ranks bit for bit
    assert np.array_equal(parts[0]["s"], parts[1]["s"]) and np.array_equal(parts[0]["V"], parts[1]["V"])
    # the sharded run reproduces the single-process run
    assert np.max(np.abs(s2 - s1) / s1) <= 1e-12
    for j in range(k):
        assert min(np.linalg.norm(V2[:, j] - V1[:, j]), np.linalg.norm(V2[:, j] + V1[:, j])) <= 1e-10
        assert min(np.linalg.norm(U2[:, j] - U1[:, j]), np.linalg.norm(U2[:, j] + U1[:, j])) <= 1e-10
    # and the true spectrum on the leading modes
    st = np.exp(-np.arange(k) / 3.0)
    assert np.max(np.abs(s2[:6] - st[:6]) / st[:6]) <= 1e-10
    # distributed CholQR2: orthonormal, same span as the sharded input
    a = _matrix(m, n)[:, :30]
    assert np.linalg.norm(Q2.T @ Q2 - np.eye(30)) <= 1e-13
    assert np.linalg.norm(a - Q2 @ (Q2.T @ a)) <= 1e-12 * np.linalg.norm(a)
    # the exchanges are the small ones: Gram and n x l partials only
    assert int(parts[0]["allreduces"]) > 0


def _rowid_worker(rank, world, port, m, k, out_dir):
    import sys

    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from _dist_numpy import row_id_rowsharded

    rs = np.random.default_rng(3)
    c = rs.standard_normal((m, k)) * np.exp(-np.arange(k) / 4.0)  # graded, distinct pivot gaps
    bounds = np.linspace(0, m, world + 1).astype(int)
    r0, r1 = bounds[rank], bounds[rank + 1]
    jr, W = row_id_rowsharded(c[r0:r1], r0, k)
    np.savez(os.path.join(out_dir, f"rid{rank}.npz"), jr=jr, W=W, c=c)
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [1, 2, 3])
def test_rowsharded_row_id_pivot_statistics_match_oracle(tmp_path, world):
    """The distributed column-pivoted QR behind the sharded CUR (csrc/dist.cu
    row_id_rowsharded, mirrored in numpy over gloo): allgathered pivot
    statistics and position bookkeeping reproduce the reference's pivots and
    interpolation matrix of id_row(C, k) for any row partition."""
    import _oracle

    m, k = 90, 12
    port = _free_port()
    mp.spawn(_rowid_worker, args=(world, port, m, k, str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(os.path.join(tmp_path, f"rid{r}.npz")) for r in range(world)]
    jr = parts[0]["jr"]
    for x in parts[1:]:
        assert np.array_equal(x["jr"], jr)  # replicated decision
    W = np.vstack([x["W"] for x in parts])
    c = parts[0]["c"]
    orc = _oracle.orc()
    ref = orc.id_column(np.asfortranarray(c.T), k)  # id_row(c, k) = id_column(c^T, k)
    assert np.array_equal(jr, ref["jc"][:k])
    assert np.max(np.abs(W - ref["v"])) <= 1e-10


def _qb_worker(rank, world, port, m, n, out_dir):
    import sys

    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from _dist_numpy import qb_rowsharded

    rs = np.random.default_rng(8)
    r = min(m, n)
    U, _ = np.linalg.qr(rs.standard_normal((m, r)))
    V, _ = np.linalg.qr(rs.standard_normal((n, r)))
    a = (U * (np.arange(r) + 1.0) ** -2) @ V.T
    bounds = np.linspace(0, m, world + 1).astype(int)
    r0, r1 = bounds[rank], bounds[rank + 1]
    Q, B, hist = qb_rowsharded(a[r0:r1], m, 8, 12, 1e-4, 1, 1, seed=5)
    np.savez(os.path.join(out_dir, f"qb{rank}.npz"), Q=Q, B=B, hist=np.array(hist), a=a)
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_rowsharded_qb_world2_matches_world1(tmp_path):
    """The row-sharded QB collective logic (csrc/dist.cu qb_blocked_rowsharded,
    mirrored in numpy over gloo): the same adaptive rank and residual history
    at world 2 as at world 1, Q orthonormal across the shards, A = QB + W."""
    m, n = 120, 90
    res = {}
    for world in (1, 2):
        d = tmp_path / f"w{world}"
        d.mkdir()
        mp.spawn(_qb_worker, args=(world, _free_port(), m, n, str(d)), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"qb{r}.npz")) for r in range(world)]
        res[world] = (np.vstack([x["Q"] for x in parts]), parts[0]["B"], parts[0]["hist"], parts[0]["a"])
        for x in parts[1:]:
            assert np.array_equal(x["B"], parts[0]["B"]) and np.array_equal(x["hist"], parts[0]["hist"])
    Q1, B1, h1, a = res[1]
    Q2, B2, h2, _ = res[2]
    assert Q1.shape == Q2.shape and len(h1) == len(h2)
    np.testing.assert_allclose(h2, h1, rtol=1e-8, atol=1e-14)
    assert np.linalg.norm(Q2.T @ Q2 - np.eye(Q2.shape[1])) <= 1e-12
    assert abs(np.linalg.norm(a - Q2 @ B2) - h2[-1]) <= 1e-10


def _qbh_worker(rank, world, port, nrb, out_dir):
    import sys

    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from _dist_numpy import qb_hierarchical_rowsharded_np

    a = _matrix(128, 48)
    base = 128 // nrb
    slabs = [a[t * base:(t + 1) * base] if t < nrb - 1 else a[t * base:] for t in range(nrb)]
    L = nrb // world
    Q, B = qb_hierarchical_rowsharded_np(slabs[rank * L:(rank + 1) * L], nrb, 4, 2, 1, seed=3)
    np.savez(os.path.join(out_dir, f"qh{rank}.npz"), Q=Q, B=B)
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world,nrb", [(2, 2), (2, 4), (4, 4)])
def test_rowsharded_hierarchical_qb_matches_single_process(tmp_path, world, nrb):
    """qb_hierarchical over ranks (csrc/dist.cu, mirrored in numpy over gloo):
    local subtree merges, the allgather of subtree-root B's and the replicated
    upper merges reproduce the single-process tree exactly."""
    from _dist_numpy import qb_hierarchical_np

    mp.spawn(_qbh_worker, args=(world, _free_port(), nrb, str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(os.path.join(tmp_path, f"qh{r}.npz")) for r in range(world)]
    Q = np.vstack([x["Q"] for x in parts])
    for x in parts[1:]:
        assert np.array_equal(x["B"], parts[0]["B"])
    a = _matrix(128, 48)
    base = 128 // nrb
    slabs = [a[t * base:(t + 1) * base] if t < nrb - 1 else a[t * base:] for t in range(nrb)]
    Qs, Bs = qb_hierarchical_np(slabs, 4, 2, 1, seed=3)
    assert np.max(np.abs(Q - Qs)) <= 1e-12 and np.max(np.abs(parts[0]["B"] - Bs)) <= 1e-12


def _tsqr_worker(rank, world, port, bounds, out_dir):
    import sys

    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import _dist_mirror as D
    from _dist_numpy import NM, NumpyBackend

    rs = np.random.default_rng(11)
    m, n, r = bounds[-1], 24, 9
    y = rs.standard_normal((m, r)) @ rs.standard_normal((r, n))  # exact rank 9 < 24 columns
    y[:, 5] = 0.0  # and an exactly zero column
    r0, r1 = bounds[rank], bounds[rank + 1]
    Q = D.orth_dist(NumpyBackend(), NM(y[r0:r1]))
    np.savez(os.path.join(out_dir, f"t{rank}.npz"), Q=Q.a, y=y)
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("bounds", [[0, 70, 140], [0, 10, 80, 150], [0, 40, 41, 90, 120]])
def test_rowsharded_orth_rank_deficient_falls_back_to_tsqr(tmp_path, bounds):
    """dist.cu's distributed orth on an exactly rank-deficient sketch (rank 9 of
    24 columns plus a zero column; csrc/dist.cu tsqr_rowsharded, mirrored):
    CholQR2 and shifted CholQR3 break down, TSQR (local QR, allgathered R
    factors, replicated QR of the compacted stack) still returns an
    orthonormal Q whose span contains the input's, including ranks that hold
    fewer rows than columns (the row-sharded path used to raise
    where the single-GPU and reference orth succeed)."""
    world = len(bounds) - 1
    port = _free_port()
    mp.spawn(_tsqr_worker, args=(world, port, bounds, str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(os.path.join(tmp_path, f"t{r}.npz")) for r in range(world)]
    Q = np.vstack([x["Q"] for x in parts])
    y = parts[0]["y"]
    assert Q.shape == y.shape
    assert np.linalg.norm(Q.T @ Q - np.eye(y.shape[1])) <= 1e-13
    assert np.linalg.norm(y - Q @ (Q.T @ y)) <= 1e-13 * np.linalg.norm(y)
