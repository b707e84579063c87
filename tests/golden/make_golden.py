"""Generate tests/golden/golden.npz from the REFERENCE itself.

Runs the unmodified reference headers (oracle/_ref/librlra_ref.so, built by
`make -C oracle ref` from /root/reference/proj/include) on small seeded
inputs and stores inputs and outputs.  The fixtures pin both the CPU oracle
restatement (bit-exact) and the product's host RNG stream; the GPU parity
tests compare against the oracle at larger sizes.

    python tests/golden/make_golden.py      # needs /root/reference (this container)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import _oracle  # noqa: E402


def main():
    ref = _oracle.ref()
    g = {}
    # --- rng stream (core/rng.hpp) -------------------------------------
    r = ref.rng(12345)
    g["rng_12345_7x3"] = ref.gaussian(7, 3, r)
    g["rng_12345_next_5x1"] = ref.gaussian(5, 1, r)
    r = ref.rng(42)
    c1 = ref.substream(r)
    c2 = ref.substream(r)
    g["rng_42_sub1_4x2"] = ref.gaussian(4, 2, c1)
    g["rng_42_sub2_4x2"] = ref.gaussian(4, 2, c2)
    # --- matmul, four cases --------------------------------------------
    rs = np.random.default_rng(2024)
    a = rs.standard_normal((9, 6))
    b = rs.standard_normal((6, 5))
    g["mm_a"], g["mm_b"] = a, b
    g["mm_nn"] = ref.matmul(a, b)
    g["mm_tn"] = ref.matmul(a, rs_b := rs.standard_normal((9, 4)), True, False)
    g["mm_tn_b"] = rs_b
    g["mm_nt"] = ref.matmul(a, rs_c := rs.standard_normal((3, 6)), False, True)
    g["mm_nt_b"] = rs_c
    # --- QR / CPQR / tri-solve KATs (tests/test_qr.cpp) -----------------
    q, rr, _ = ref.compact_qr(np.array([[3.0], [4.0]]))
    g["orth_34"] = q
    x = rs.standard_normal((20, 6))
    g["qr_in"] = x
    g["qr_q"], g["qr_r"], _ = ref.compact_qr(x)
    f = ref.pivoted_qr(np.diag([3.0, 2.0, 1.0]), 2)
    g["cpqr_diag_perm"] = f["perm"]
    g["cpqr_diag_res"] = np.array([f["residual"]])
    x = rs.standard_normal((12, 15))
    g["cpqr_in"] = x
    f = ref.pivoted_qr(x, 8)
    g["cpqr_perm"], g["cpqr_s1"], g["cpqr_res"] = f["perm"], f["s1"], np.array([f["residual"]])
    t, cl = ref.upper_tri_solve(np.array([[1e8, 0.0], [0.0, 1e-8]]), np.array([[1.0], [1.0]]))
    g["trisolve_clamp"] = t
    # --- jacobi ---------------------------------------------------------
    u, s, v = ref.small_svd(np.diag([2.0, -3.0]))
    g["svd_diag_sigma"] = s
    x = rs.standard_normal((10, 7))
    g["svd_in"] = x
    g["svd_u"], g["svd_s"], g["svd_v"] = ref.small_svd(x)
    # --- algorithms on a small spectral matrix --------------------------
    m, n = 60, 40
    U, _ = np.linalg.qr(rs.standard_normal((m, n)))
    V, _ = np.linalg.qr(rs.standard_normal((n, n)))
    A = np.asfortranarray((U * np.exp(-np.arange(n) / 5.0)) @ V.T)
    g["A"] = A
    for var, name in [(0, "v2"), (1, "v1"), (2, "basic")]:
        u, s, v = ref.rsvd(A, 8, 4, 2, 1, ref.rng(12345), var)
        g[f"rsvd_{name}_u"], g[f"rsvd_{name}_s"], g[f"rsvd_{name}_v"] = u, s, v
    f = ref.qb_blocked(A, 5, 6, 1e-3, 1, 1, ref.rng(12345))
    g["qb_q"], g["qb_b"], g["qb_hist"] = f["q"], f["b"], f["history"]
    g["qb_ell"] = np.array([f["ell"]])
    u, s, v = ref.svd_from_qb(f["q"], f["b"], 0, 0)
    g["svdqb_s"] = s
    f = ref.id_rand(A, 10, 5, 2, 1, ref.rng(12345))
    g["idrand_jc"], g["idrand_v"], g["idrand_res"] = f["jc"], f["v"], np.array([f["qr_residual"]])
    f = ref.cur_rand(A, 10, 5, 2, 1, ref.rng(12345))
    for key in ("jc", "jr", "c", "u", "r"):
        g[f"cur_{key}"] = f[key]
    g["cur_res"] = np.array([f["residual"], f["qr_residual"]])
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **g)
    print(f"wrote {len(g)} arrays")


if __name__ == "__main__":
    main()
