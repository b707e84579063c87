"""Python restatement of the row-sharded orchestration of csrc/dist.cu
(TEST INFRASTRUCTURE ONLY; not part of the product package).

tests/test_dist_gloo.py runs it at world size 2-4 over gloo on CPU with the
numpy stand-in backend of tests/_dist_numpy.py, where no GPU exists, to check
the collective logic (which sums are exchanged, which factors are replicated)
against the single-process oracle.  The product path is the C++ driver
(csrc/dist.cu), exercised at world sizes 2-4 on one GPU by
tests/test_gpu_dist_ranks.py through host-staged collectives.
"""
from paper_1502_05366_b200 import DimensionError, RlraError

PIVOT_FLOOR = 1e-12  # same breakdown test as the single-GPU CholQR2 (qr.cu)


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
    """dist.cu shifted_cholqr3_rowsharded; TSQR when it breaks down."""
    m_tot_n = be.allreduce_scalar(float(Y.rows))
    fro2 = be.allreduce_scalar(be.fro2(Y))
    n = Y.cols
    if not fro2 > 0.0:
        return tsqr_dist(be, Y)
    shift = 11.0 * (m_tot_n * n + n * (n + 1)) * 1.1102230246251565e-16 * fro2
    G = be.allreduce(be.gram(Y))
    be.add_diag(G, shift)
    f = be.chol_inv(G, 0.0)
    if f is None:
        return tsqr_dist(be, Y)
    Y1 = be.trmm(Y, f[1])
    for _ in range(2):
        G = be.allreduce(be.gram(Y1))
        f = be.chol_inv(G, PIVOT_FLOOR)
        if f is None:
            return tsqr_dist(be, Y)
        Y1 = be.trmm(Y1, f[1])
    return Y1


def tsqr_dist(be, Y):
    """dist.cu tsqr_rowsharded: local QR, allgather of the (padded) R
    factors, replicated QR of the compacted stack (rank r contributes
    min(m_r, n) rows), Y_g <- Q_g Qhat_g (or Qhat_g itself when m_g < n)."""
    import numpy as np

    from _dist_numpy import NM

    mg, n = Y.rows, Y.cols
    rows = [int(x[0, 0]) for x in be.allgather(NM(np.array([[float(mg)]])))]
    Rg = np.zeros((n, n))
    Qg = None
    if mg >= n:
        Qg, R = be.qr_local(Y)
        Rg[:] = R.a
    elif mg > 0:
        Rg[:mg] = Y.a
    allR = be.allgather(NM(Rg))
    take = [min(r, n) for r in rows]
    S = np.vstack([allR[r][:take[r]] for r in range(len(rows))])
    if S.shape[0] < n:
        raise RlraError(f"tsqr: {S.shape[0]} stacked rows for {n} columns")
    Qh, _ = be.qr_local(NM(S))
    off = sum(take[:be.rank])
    if mg >= n:
        return be.matmul(Qg, NM(Qh.a[off:off + n]))
    return NM(Qh.a[off:off + mg])


def check_sample_rank(k, p, m, n):
    
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


