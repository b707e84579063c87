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
        self.rank = dist.get_rank() if dist.is_initialized() else 0
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

    def allgather(self, X):
        """list of every rank's X (same shape on every rank)"""
        if self.world <= 1:
            return [np.array(X.a)]
        t = torch.from_numpy(np.ascontiguousarray(X.a))
        outs = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(outs, t)
        return [o.numpy() for o in outs]

    def allreduce_scalar(self, x):
        if self.world <= 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t)
        return float(t.item())


# ---------------------------------------------------------------------------
# numpy mirror of csrc/dist.cu row_id_rowsharded (the distributed column-
# pivoted QR of C^T whose columns -- the rows of C -- are sharded): the same
# per-step record allgather, winner rule, position bookkeeping, allreduced
# pivot column and reflector/downdate arithmetic, with gloo collectives.
def _better(v, p, bv, bp):
    return v > bv or (v == bv and p < bp)


def row_id_rowsharded(Cg, row0, k):
    """Returns (jr: k global pivot rows, W_g: this rank's rows of W)."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    X = np.array(Cg.T, dtype=np.float64, order="F")  # k x mg
    mg = X.shape[1]
    pos = np.arange(row0, row0 + mg, dtype=np.float64)
    cn = (X * X).sum(0)
    rn = cn.copy()
    S11 = np.zeros((k, k))
    jr = np.zeros(k, dtype=np.int64)
    for f in range(k):
        bv, bp, bj = -np.inf, np.inf, -1
        for j in range(mg):
            if pos[j] >= f and _better(cn[j], pos[j], bv, bp):
                bv, bp, bj = cn[j], pos[j], j
        rec = torch.tensor([bv if bj >= 0 else -np.inf, bp, row0 + bj if bj >= 0 else -1.0, float(bj)],
                           dtype=torch.float64)
        recs = [torch.zeros(4, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(recs, rec) if world > 1 else recs.__setitem__(0, rec)
        wv, wp, wg, wj, wr = -np.inf, np.inf, -1, -1, -1
        for r, q in enumerate(recs):
            q = q.numpy()
            if q[3] >= 0 and _better(q[0], q[1], wv, wp):
                wv, wp, wg, wj, wr = q[0], q[1], q[2], int(q[3]), r
        jr[f] = int(wg)
        me = dist.get_rank() if world > 1 else 0
        pc = torch.tensor(X[:, wj] if wr == me else np.zeros(k), dtype=torch.float64)
        if world > 1:
            dist.all_reduce(pc)
        pc = pc.numpy()
        pos[pos == f] = wp
        if wr == me:
            pos[wj] = f
        norm2 = float(np.sum(pc[f:] ** 2))
        x1, norm = pc[f], np.sqrt(norm2)
        zero = norm < 1e-300
        alpha = -norm if x1 >= 0 else norm
        beta = 0.0 if zero else 2.0 / (2.0 * (norm2 - alpha * x1))
        alpha = 0.0 if zero else alpha
        v = np.zeros(k)
        v[f] = pc[f] - (alpha if beta != 0.0 else 0.0)
        v[f + 1:] = pc[f + 1:]
        S11[:f, f] = pc[:f]
        S11[f, f] = alpha
        for j in range(mg):
            if wr == me and j == wj:
                X[f, j] = alpha
                X[f + 1:, j] = 0.0
                continue
            if pos[j] <= f:
                continue
            if beta != 0.0:
                X[f:, j] -= beta * float(v[f:] @ X[f:, j]) * v[f:]
            c = cn[j] - X[f, j] ** 2
            if c < 1e-6 * rn[j]:
                c = float(np.sum(X[f + 1:, j] ** 2))
                rn[j] = c
            cn[j] = c
    sg = np.where(np.diag(S11) < 0, -1.0, 1.0)
    S11 = S11 * sg[:, None]
    X = X * sg[:, None]
    T = np.linalg.solve(S11, X) if mg else X
    if np.max(np.abs(np.diag(S11))) / np.min(np.abs(np.diag(S11))) > 1e12:
        T = np.clip(T, -1e4, 1e4)
    W = np.zeros((mg, k))
    for j in range(mg):
        W[j] = np.eye(k)[int(pos[j])] if pos[j] < k else T[:, j]
    return jr, W


# numpy mirror of csrc/dist.cu qb_blocked_rowsharded (qb.hpp:98-142 on a
# row-sharded W): the collectives are the b x b Gram (inside the distributed
# QR), the n x b power partials, the l x b reorth projection, B_i and ||W||^2.
def _allreduce(x):
    if dist.is_initialized() and dist.get_world_size() > 1:
        t = torch.from_numpy(np.ascontiguousarray(x))
        dist.all_reduce(t)
        return t.numpy()
    return x


def _orth_rows(Y):
    """CholQR2 of the row-sharded Y (Gram allreduce, replicated Cholesky)."""
    for _ in range(2):
        G = _allreduce(Y.T @ Y)
        R = np.linalg.cholesky(G).T
        Y = np.linalg.solve(R.T, Y.T).T
    return Y


def qb_rowsharded(Wg, m_total, b, M, tol, q, reorth, seed):
    Wg = np.array(Wg, dtype=np.float64, order="F")
    n = Wg.shape[1]
    rmax = min(m_total, n)
    Q = np.zeros((Wg.shape[0], 0))
    B = np.zeros((0, n))
    hist = []
    for i in range(1, M + 1):
        width = min(b, rmax - Q.shape[1])
        if width < 1:
            break
        Om = omega_rows(seed, i, 0, n, width)  # the same n x b draw on every rank
        Qi = _orth_rows(Wg @ Om)
        for _ in range(q):
            Z = np.linalg.qr(_allreduce(Wg.T @ Qi))[0]
            Qi = _orth_rows(Wg @ Z)
        if i % reorth == 0:
            if Q.shape[1]:
                Qi = Qi - Q @ _allreduce(Q.T @ Qi)
            Qi = _orth_rows(Qi)
        Bi = _allreduce(Qi.T @ Wg)
        Wg = Wg - Qi @ Bi
        Q = np.hstack([Q, Qi])
        B = np.vstack([B, Bi])
        r = float(np.sqrt(_allreduce(np.array([np.sum(Wg * Wg)]))[0]))
        hist.append(r)
        if tol > 0 and r < tol:
            break
    return Q, B, hist


# numpy mirror of csrc/dist.cu qb_hierarchical_rowsharded: leaves and the
# rank's subtree locally, allgather of the subtree-root B's, replicated upper
# merges, Q lifted through this rank's path.  Fixed-rank QB with counter-based
# Omega per (node, block) so the single-process and sharded runs draw alike.
def _qb_fixed(W, b, M, q, node, seed):
    n = W.shape[1]
    Q = np.zeros((W.shape[0], 0))
    B = np.zeros((0, n))
    for i in range(M):
        Om = omega_rows(seed, (node << 16) | i, 0, n, b)
        Qi = np.linalg.qr(W @ Om)[0]
        for _ in range(q):
            Qi = np.linalg.qr(W @ np.linalg.qr(W.T @ Qi)[0])[0]
        if Q.shape[1]:
            Qi = np.linalg.qr(Qi - Q @ (Q.T @ Qi))[0]
        Bi = Qi.T @ W
        W = W - Qi @ Bi
        Q, B = np.hstack([Q, Qi]), np.vstack([B, Bi])
    return Q, B


def qb_hierarchical_np(slabs, b, M, q, seed):
    """Single-process reference: slabs is the list of row slabs."""
    nrb = len(slabs)
    nodes = [_qb_fixed(s, b, M, q, t, seed) for t, s in enumerate(slabs)]
    mid = nrb
    while len(nodes) > 1:
        nxt = []
        for t in range(0, len(nodes), 2):
            (ql, bl), (qr, br) = nodes[t], nodes[t + 1]
            qm, bm = _qb_fixed(np.vstack([bl, br]), b, M, q, mid, seed)
            mid += 1
            r = bl.shape[0]
            nxt.append((np.vstack([ql @ qm[:r], qr @ qm[r:]]), bm))
        nodes = nxt
    return nodes[0]


def qb_hierarchical_rowsharded_np(my_slabs, nrb, b, M, q, seed):
    world, g = dist.get_world_size(), dist.get_rank()
    L = len(my_slabs)
    rank = b * M

    def merge_id(lv, pi):
        idx, cnt = nrb, nrb
        for _ in range(lv):
            cnt //= 2
            idx += cnt
        return idx + pi

    nodes = [_qb_fixed(s, b, M, q, g * L + t, seed) for t, s in enumerate(my_slabs)]
    lv = 0
    while len(nodes) > 1:
        nxt = []
        for t in range(0, len(nodes), 2):
            (ql, bl), (qr, br) = nodes[t], nodes[t + 1]
            qm, bm = _qb_fixed(np.vstack([bl, br]), b, M, q, merge_id(lv, g * (len(nodes) // 2) + t // 2), seed)
            nxt.append((np.vstack([ql @ qm[:rank], qr @ qm[rank:]]), bm))
        nodes = nxt
        lv += 1
    Bs = [torch.zeros(rank, nodes[0][1].shape[1], dtype=torch.float64) for _ in range(world)]
    dist.all_gather(Bs, torch.from_numpy(np.ascontiguousarray(nodes[0][1])))
    up = [x.numpy() for x in Bs]
    T = np.eye(rank)
    pos = g
    while len(up) > 1:
        nxt = []
        for t in range(0, len(up), 2):
            qm, bm = _qb_fixed(np.vstack([up[t], up[t + 1]]), b, M, q, merge_id(lv, t // 2), seed)
            if t == (pos & ~1):
                T = T @ (qm[rank:] if pos & 1 else qm[:rank])
            nxt.append(bm)
        up = nxt
        pos >>= 1
        lv += 1
    return nodes[0][0] @ T, up[0]
