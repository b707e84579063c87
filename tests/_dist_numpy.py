"""numpy stand-in for dist.GpuBackend (TEST INFRASTRUCTURE ONLY).

Lets tests/test_dist_gloo.py run the row-sharded orchestration of
paper_1502_05366_b200/dist.py at world size 2 over gloo on CPU, where no GPU
exists.  Omega is a counter-based draw per (seed, draw, global row) so every
rank sees the same Omega rows, like the engine's Philox.
"""
import numpy as np
import torch
import torch.distributed as dist


class NM:
    def __init__(self, a):
        self.a = np.asfortranarray(a)

    @property
    def rows(self):
        return self.a.shape[0]

    @property
    def cols(self):
        return self.a.shape[1]

    def cols_view(self, k):
        return NM(self.a[:, :k])


class OmegaSeed:
    def __init__(self, seed):
        self.seed = seed


def omega_rows(seed, draw, row0, rows, l):
    return np.stack([np.random.default_rng([seed, draw, row0 + i]).standard_normal(l)
                     for i in range(rows)]) if rows else np.zeros((0, l))


class NumpyBackend:
    def __init__(self):
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.allreduces = 0

    def new(self, rows, cols):
        return NM(np.zeros((rows, cols)))

    def wrap(self, a, rows, cols):
        return NM(a)

    def sketch(self, A, l, omega, draw, row0, trans):
        if trans:
            return NM(A.a.T @ omega_rows(omega.seed, draw, row0, A.rows, l))
        return NM(A.a @ omega_rows(omega.seed, draw, 0, A.cols, l))

    def matmul(self, A, B, ta=False, tb=False):
        a = A.a.T if ta else A.a
        b = B.a.T if tb else B.a
        return NM(a @ b)

    def gram(self, Y):
        return NM(Y.a.T @ Y.a)

    def chol_inv(self, G, floor):
        g = G.a
        try:
            L = np.linalg.cholesky(g)
        except np.linalg.LinAlgError:
            return None
        R = L.T
        if np.any(np.diag(R) ** 2 < floor * np.diag(g)):
            return None
        Ri = np.linalg.solve(R, np.eye(R.shape[0]))
        return NM(np.triu(R)), NM(np.triu(Ri))

    def trmm(self, Y, T):
        return NM(Y.a @ T.a)

    def add_diag(self, G, s):
        G.a[np.diag_indices_from(G.a)] += s

    def fro2(self, Y):
        return float(np.sum(Y.a ** 2))

    def qr_local(self, Y):
        q, r = np.linalg.qr(Y.a)
        sg = np.where(np.diag(r) < 0, -1.0, 1.0)
        return NM(q * sg), NM(r * sg[:, None])

    def svd_local(self, Rm):
        u, s, vt = np.linalg.svd(Rm.a)
        return NM(u), NM(s[:, None]), NM(vt.T)

    def allreduce(self, X):
        if self.world > 1:
            t = torch.from_numpy(np.ascontiguousarray(X.a))
            dist.all_reduce(t)
            self.allreduces += 1
            return NM(t.numpy())
        return X

    def allreduce_scalar(self, x):
        if self.world <= 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t)
        return float(t.item())
