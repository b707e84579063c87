"""Row-sharded multi-GPU randomized SVD (BASELINE north_star).

A (m x n) is split by rows across the ranks of a torch.distributed group (one
process per GPU, NCCL over NVLink).  Every product with A is local to a shard;
the exchanges are the small ones north_star names:

  * Y_g = A_g Omega                         local (Philox Omega is the same on
                                            every rank: its counter is the
                                            global (row, column))
  * orth(Y), Y row-sharded                  CholQR2 with an allreduce of the
                                            l x l Gram per pass; the Cholesky
                                            and R^{-1} are replicated
  * Z = A^T Y = sum_g A_g^T Y_g             allreduce of n x l
  * Bt = A^T Q                              allreduce of n x l (the partial
                                            Q^T A of north_star)
  * QR(Bt), Jacobi SVD of R-hat             replicated
  * U_g = Q_g Vhat                          local

The algorithm is the reference's rsvd_v2 (rsvd.hpp:154-160, sketch.hpp:44-60)
with the same Omega; only the association order of the sums changes.

The product path is the C++ driver (csrc/dist.cu, C-ABI rlra_rsvd_rowsharded)
with its own NCCL communicator: `NcclComm` below creates it (rank 0's
unique id travels over the torch.distributed group) and `rsvd_v2_native`
calls it.  The Python orchestration further down restates the same algorithm
against a small backend interface so the collective logic also runs, in the
test-suite, on a numpy stand-in over gloo (tests/_dist_numpy.py) at world
size 2 without GPUs; `GpuBackend` runs that restatement on the engine's
shard primitives.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import RlraError

PIVOT_FLOOR = 1e-12  # same breakdown test as the single-GPU CholQR2 (qr.cu)


# ---------------------------------------------------------------- backend ---
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

    def cols_view(self, k):
        return DM(self.t[: self.rows * k], self.rows, k)


class GpuBackend:
    """Per-shard steps on the CUDA engine; collectives through torch.distributed."""

    def __init__(self, eng, group=None):
        import torch
        import torch.distributed as dist

        self.torch = torch
        self.dist = dist
        self.eng = eng
        self.dev = torch.device("cuda", eng.device)
        self.group = group
        self.comm = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if self.comm else 1
        self.rank = dist.get_rank(group) if self.comm else 0

    def new(self, rows, cols):
        return DM(self.torch.empty(max(rows * cols, 1), dtype=self.torch.float64, device=self.dev),
                  rows, cols)

    def wrap(self, t, rows, cols):
        return DM(t, rows, cols)

    def sketch(self, A, l, omega, draw, row0, trans):
        Y = self.new(A.cols if trans else A.rows, l)
        self.eng.device_sketch(trans, A.ptr, A.rows, A.cols, A.ld, l, omega, draw, row0, Y.ptr, Y.ld)
        return Y

    def matmul(self, A, B, ta=False, tb=False):
        m = A.cols if ta else A.rows
        n = B.rows if tb else B.cols
        Cm = self.new(m, n)
        self.eng.device_matmul(ta, tb, A.ptr, A.rows, A.cols, A.ld, B.ptr, B.rows, B.cols, B.ld,
                               Cm.ptr, Cm.ld)
        return Cm

    def gram(self, Y):
        G = self.new(Y.cols, Y.cols)
        self.eng.device_gram(Y.ptr, Y.rows, Y.cols, Y.ld, G.ptr, G.ld)
        return G

    def chol_inv(self, G, floor):
        R, Ri = self.new(G.rows, G.rows), self.new(G.rows, G.rows)
        ok = self.eng.device_chol_inv(G.ptr, G.rows, G.ld, floor, R.ptr, R.ld, Ri.ptr, Ri.ld)
        return (R, Ri) if ok else None

    def trmm(self, Y, T):
        O = self.new(Y.rows, Y.cols)
        self.eng.device_trmm_right_upper(Y.ptr, Y.rows, Y.cols, Y.ld, T.ptr, T.ld, O.ptr, O.ld)
        return O

    def add_diag(self, G, s):
        self.torch.diagonal(G.t[: G.rows * G.cols].view(G.cols, G.rows)).add_(s)
        self.torch.cuda.synchronize(self.dev)

    def fro2(self, Y):
        return float(self.torch.sum(Y.t[: Y.rows * Y.cols] ** 2))

    def qr_local(self, Y):
        Q, R = self.new(Y.rows, Y.cols), self.new(Y.cols, Y.cols)
        self.eng.device_compact_qr(Y.ptr, Y.rows, Y.cols, Y.ld, Q.ptr, Q.ld, R.ptr, R.ld)
        return Q, R

    def svd_local(self, Rm):
        r = min(Rm.rows, Rm.cols)
        U, V, s = self.new(Rm.rows, r), self.new(Rm.cols, r), self.new(r, 1)
        self.eng.device_small_svd(Rm.ptr, Rm.rows, Rm.cols, Rm.ld, U.ptr, U.ld, s.ptr, V.ptr, V.ld)
        return U, s, V

    def allreduce(self, X):
        if self.comm:
            self.eng.synchronize()
            self.dist.all_reduce(X.t[: X.rows * X.cols], group=self.group)
            self.torch.cuda.synchronize(self.dev)
        return X

    def allreduce_scalar(self, x):
        if not self.comm:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, group=self.group)
        return float(t.item())


# ------------------------------------------------ native C++/NCCL driver --
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


# ----------------------------------------------------------- orchestration --
def orth_dist(be, Y, span_only=False):
    """CholQR2 of the row-sharded Y (qr.cu's policy, distributed): Gram
    allreduce -> replicated Cholesky/R^{-1} -> local Y R^{-1}; one pass when
    only the span is consumed.  Shifted CholQR3 when the Gram is too
    ill-conditioned.  Returns the local block of Q."""
    G = be.allreduce(be.gram(Y))
    f = be.chol_inv(G, PIVOT_FLOOR)
    if f is None:
        return _shifted_cholqr3_dist(be, Y)
    Y1 = be.trmm(Y, f[1])
    if span_only:
        return Y1
    G2 = be.allreduce(be.gram(Y1))
    f2 = be.chol_inv(G2, PIVOT_FLOOR)
    if f2 is None:
        return _shifted_cholqr3_dist(be, Y)
    return be.trmm(Y1, f2[1])


def _shifted_cholqr3_dist(be, Y):
    m_tot_n = be.allreduce_scalar(float(Y.rows))
    fro2 = be.allreduce_scalar(be.fro2(Y))
    n = Y.cols
    shift = 11.0 * (m_tot_n * n + n * (n + 1)) * 1.1102230246251565e-16 * fro2
    G = be.allreduce(be.gram(Y))
    be.add_diag(G, shift)
    f = be.chol_inv(G, 0.0)
    if f is None:
        raise RlraError("distributed orth: shifted CholQR3 broke down (rank-deficient sketch)")
    Y1 = be.trmm(Y, f[1])
    for _ in range(2):
        G = be.allreduce(be.gram(Y1))
        f = be.chol_inv(G, PIVOT_FLOOR)
        if f is None:
            raise RlraError("distributed orth: sketch is rank deficient to working precision")
        Y1 = be.trmm(Y1, f[1])
    return Y1


def check_sample_rank(k, p, m, n):
    from . import DimensionError

    if k < 1:
        raise DimensionError(f"rank k must be >= 1 (got {k})")
    if p < 0:
        raise DimensionError(f"oversampling p must be >= 0 (got {p})")
    if k + p > min(m, n):
        raise DimensionError(f"k + p = {k + p} exceeds min(m,n) = {min(m, n)}")


def rsvd_v2_rowsharded(be, A, m_total, k, p, q, s, omega):
    """rsvd_v2 on a row-sharded A.  A is this rank's m_g x n row block.
    Returns (U_g, sigma, V): U row-sharded like A, sigma and V replicated."""
    n = A.cols
    l = k + p
    check_sample_rank(k, p, m_total, n)
    if q < 0 or s < 1:
        from . import DimensionError
        raise DimensionError(f"sample_right: q={q}, s={s} out of range")
    Y = be.sketch(A, l, omega, 0, 0, False)               # sketch.hpp:51-52
    for j in range(1, q + 1):                              # sketch.hpp:53-58
        if (2 * j - 2) % s == 0:
            Y = orth_dist(be, Y, span_only=True)
        Z = be.allreduce(be.matmul(A, Y, ta=True))
        if (2 * j - 1) % s == 0:
            Z = be.qr_local(Z)[0]
        Y = be.matmul(A, Z)
    Q = orth_dist(be, Y)                                   # rsvd.hpp:157
    Bt = be.allreduce(be.matmul(A, Q, ta=True))            # rsvd.hpp:158
    Qh, Rh = be.qr_local(Bt)                               # rsvd.hpp:148
    Uh, sg, Vh = be.svd_local(Rh)
    U = be.matmul(Q, Vh.cols_view(k))
    V = be.matmul(Qh, Uh.cols_view(k))
    return U, sg, V


def gen_test_matrix_rowsharded(be, n, row0, m_local, sigma, seed):
    """Rows [row0, row0 + m_local) of A = U diag(sigma) V^T, U and V
    orthonormalised Philox Gaussians; U is orthonormalised across ranks with
    the distributed CholQR2, V (n x r) is identical on every rank."""
    r = len(sigma)
    U = be.new(m_local, r)
    V = be.new(n, r)
    be.eng.device_gaussian_philox(m_local, r, seed, 101, row0, U.ptr, U.ld)
    be.eng.device_gaussian_philox(n, r, seed, 102, 0, V.ptr, V.ld)
    U = orth_dist(be, U)
    V = be.qr_local(V)[0]
    import torch
    s = torch.as_tensor(np.asarray(sigma, dtype=np.float64), device=be.dev)
    U.t[: m_local * r].view(r, m_local).mul_(s.view(r, 1))
    A = be.matmul(U, V, tb=True)
    return A, s
