"""Row-sharded multi-GPU path (BASELINE north_star): the
launch-side helpers around the C++ driver (csrc/dist.cu).

A (m x n) is split by rows across the ranks (one process per GPU, or ranks as
threads).  Every product with A is local to a shard; the exchanges are the
small ones north_star names (allreduce of the l x l Grams and of the n x l
partials A_g^T Y_g / A_g^T Q_g, allgathered TSQR R factors and pivot
statistics).  The orchestration is C++ (rlra_*_rowsharded); this module only
builds its communicators:

  * ``NcclComm``   NCCL over NVLink, one process per GPU: rank 0's unique id
                   travels over a torch.distributed group.
  * ``HostComm``   host-staged collectives over a torch.distributed group
                   (gloo): the driver copies each exchanged buffer to pinned
                   host memory and back, so no kernel waits on another rank;
                   ``share_gpu=True`` adds a file-lock GPU token so several
                   ranks may share one GPU.
  * ``LocalGroup`` (package root) ranks as threads of one process.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import HostCollectives


@dataclass
class DM:
    """Column-major device matrix: flat float64 CUDA tensor, ld == rows."""
    t: object
    rows: int
    cols: int

    @property
    def ptr(self):
        return self.t.data_ptr()

    @property
    def ld(self):
        return max(1, self.rows)


class NcclComm:
    """The engine's NCCL communicator (rlra_comm) for the ranks of a
    torch.distributed group: rank 0 draws the unique id, the group broadcasts
    it, every rank joins."""

    def __init__(self, eng, group=None):
        import torch
        import torch.distributed as dist

        self.eng = eng
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = eng.comm_unique_id() if self.rank == 0 else bytes(128)
        if self.world > 1:
            dev = torch.device("cuda", eng.device) if dist.get_backend(group) == "nccl" else torch.device("cpu")
            t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
            dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
            uid = bytes(t.cpu().tolist())
        self.handle = eng.comm_create(uid, self.world, self.rank)

    def close(self):
        if self.handle:
            self.eng.comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _FileToken:
    """A GPU token shared by processes: an exclusive flock on a lock file."""

    def __init__(self, path):
        self.fd = os.open(path, os.O_CREAT | os.O_RDWR, 0o666)

    def acquire(self):
        import fcntl
        fcntl.flock(self.fd, fcntl.LOCK_EX)

    def release(self):
        import fcntl
        fcntl.flock(self.fd, fcntl.LOCK_UN)

    def close(self):
        if self.fd >= 0:
            os.close(self.fd)
            self.fd = -1


class HostComm:
    """rlra_comm over host-staged collectives of a torch.distributed group
    (gloo): allreduce_sum / allgather of CPU tensors.  With ``share_gpu`` the
    ranks take turns on the GPU (a file-lock token), so several ranks may
    run on one device without any kernel waiting on another rank's."""

    def __init__(self, eng, group=None, share_gpu=False, lock_path=None):
        import torch
        import torch.distributed as dist

        self.eng = eng
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self._tok = None
        if share_gpu:
            self._tok = _FileToken(lock_path or f"/tmp/rlra_gpu{eng.device}_{os.getppid()}.lock")

        def allreduce_sum(buf):
            t = torch.from_numpy(buf)
            dist.all_reduce(t, group=group)

        def allgather(send, recv):
            n = send.shape[0]
            outs = [torch.from_numpy(recv[r * n:(r + 1) * n]) for r in range(self.world)]
            dist.all_gather(outs, torch.from_numpy(send.copy()), group=group)

        self.coll = HostCollectives(allreduce_sum, allgather,
                                    self._tok.acquire if self._tok else None,
                                    self._tok.release if self._tok else None)
        self.handle = eng.comm_create_host(self.world, self.rank, self.coll)

    def close(self):
        if self.handle:
            self.eng.comm_destroy(self.handle)
            self.handle = None
        if self._tok:
            self._tok.close()
            self._tok = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def rsvd_v2_native(comm, A, m_total, k, p, q, s, omega):
    """rsvd_v2 on this rank's row block A (DM, m_g x n) through the C++
    driver; returns (U_g, sigma, V) as DMs (U row-sharded, sigma and V
    replicated)."""
    import torch

    eng = comm.eng
    n = A.cols
    dev = torch.device("cuda", eng.device)
    U = DM(torch.empty(max(A.rows * k, 1), dtype=torch.float64, device=dev), A.rows, k)
    S = DM(torch.empty(k, dtype=torch.float64, device=dev), k, 1)
    V = DM(torch.empty(n * k, dtype=torch.float64, device=dev), n, k)
    eng.device_rsvd_rowsharded(comm.handle, A.ptr, A.rows, n, A.ld, m_total, k, p, q, s, omega, U.ptr, U.ld,
                               S.ptr, V.ptr, V.ld)
    return U, S, V


def gen_test_matrix_rowsharded(comm, n, row0, m_local, m_total, sigma, seed, noise=0.0):
    """Rows [row0, row0 + m_local) of A = U diag(sigma) V^T (+ noise G) as a DM,
    through rlra_gen_test_matrix_rowsharded (U orthonormalised across the
    ranks); returns (A_g, sigma) with sigma a device tensor."""
    import torch

    eng = comm.eng
    dev = torch.device("cuda", eng.device)
    sigma = np.ascontiguousarray(sigma, dtype=np.float64)
    A = torch.empty(max(m_local * n, 1), dtype=torch.float64, device=dev)
    eng.device_gen_test_matrix_rowsharded(comm.handle, row0, m_local, m_total, n, sigma, seed, noise,
                                          A.data_ptr(), max(1, m_local))
    return DM(A, m_local, n), torch.as_tensor(sigma, device=dev)
