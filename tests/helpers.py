"""Shared test helpers: seeded test matrices and comparisons (test-only)."""
import numpy as np


def rel_fro(x, y):
    y = np.asarray(y)
    d = np.linalg.norm(np.asarray(x) - y)
    n = np.linalg.norm(y)
    return d / n if n > 0 else d


def make_test_matrix(m, n, sigma, seed):
    """A = U diag(sigma) V^T with U, V orthonormalised seeded Gaussians
    (the reference's gen_test_matrix recipe, testmat.hpp:65-74, built with
    numpy's QR for speed; only its spectrum matters to the tests)."""
    rs = np.random.default_rng(seed)
    r = len(sigma)
    U, _ = np.linalg.qr(rs.standard_normal((m, r)))
    V, _ = np.linalg.qr(rs.standard_normal((n, r)))
    return np.asfortranarray((U * np.asarray(sigma)) @ V.T)


def exact_rank(m, n, r, seed):
    rs = np.random.default_rng(seed)
    return np.asfortranarray(rs.standard_normal((m, r)) @ rs.standard_normal((r, n)))


def orthonormality_defect(q):
    q = np.asarray(q)
    return np.linalg.norm(q.T @ q - np.eye(q.shape[1]))


def reconstruct(u, s, v):
    return (np.asarray(u) * np.asarray(s)) @ np.asarray(v).T


def match_columns_up_to_sign(x, y):
    """max over columns of min(||x_j - y_j||, ||x_j + y_j||)."""
    x, y = np.asarray(x), np.asarray(y)
    return max(min(np.linalg.norm(x[:, j] - y[:, j]), np.linalg.norm(x[:, j] + y[:, j]))
               for j in range(x.shape[1])) if x.shape[1] else 0.0
