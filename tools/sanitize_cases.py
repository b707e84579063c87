"""Small invocations of every cooperative / barrier-heavy kernel of the path
for compute-sanitizer (racecheck, synccheck, memcheck): one case per process
(the kernel choice of small_svd is read once per process).  Host API only (no
torch), so the sanitizer sees just the engine's kernels.
Usage: python tools/sanitize_cases.py <case>   (cases: see CASES)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_1502_05366_b200 as R


def mat(m, n, r, seed, decay=10.0):
    rs = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rs.standard_normal((m, r)))
    V, _ = np.linalg.qr(rs.standard_normal((n, r)))
    return np.asfortranarray((U * np.exp(-np.arange(r) / decay)) @ V.T)


def rsvd(eng):  # sketch GEMM (TMA), CholQR2 (chol_inv_coop), bgram Jacobi, lift
    u, s, v = eng.rsvd_v2(mat(1500, 900, 300, 1), 60, 10, 2, 1, rng=R.Rng(1))
    assert s[0] > 0


def idcur(eng):  # id_rand (cpqr_step_kernel, trisolve), cur_rand (row ID, linkage)
    a = mat(700, 500, 200, 2)
    eng.id_rand(a, 50, 10, 2, 1, rng=R.Rng(2))
    eng.cur_rand(a, 50, 10, 2, 1, rng=R.Rng(3))


def qb(eng):  # blocked QB: EPI_RESID GEMM, reorth, span orth
    eng.qb_blocked(mat(600, 500, 300, 3, 20.0), 16, 20, 1e-6, 1, 1, rng=R.Rng(4))


def chol(eng):  # one-launch cooperative Cholesky at l > 64 (several block steps), Householder fallback
    a = mat(4000, 300, 300, 5, 60.0)
    eng.orth(a)
    b = mat(800, 120, 40, 6)  # rank 40 < 120 columns: CholQR breaks down -> Householder
    eng.orth(b)


def sgram(eng):  # streaming Gram block Jacobi (C2 kernel) on a small R-hat
    eng.small_svd(np.triu(mat(240, 240, 240, 7, 40.0)))


def gemm(eng):  # TMA GEMM NN / TN / split-K shapes
    rs = np.random.default_rng(8)
    a, b = rs.standard_normal((700, 600)), rs.standard_normal((600, 300))
    eng.matmul(a, b)
    eng.matmul(rs.standard_normal((5000, 300)), rs.standard_normal((5000, 260)), trans_a=True)


CASES = dict(rsvd=rsvd, idcur=idcur, qb=qb, chol=chol, sgram=sgram, gemm=gemm)

if __name__ == "__main__":
    name = sys.argv[1]
    if name == "sgram":
        os.environ["RLRA_SVD_KERNEL"] = "sgram"
    eng = R.Engine(0)
    CASES[name](eng)
    eng.synchronize()
    print(f"case {name} ok", flush=True)
