"""rlra-b200: B200-native engine for the reference's randomized low-rank
factorization path (RSVDPACK-class, arXiv:1502.05366).

This module is the ctypes binding a Python user (and the test-suite and
bench.py) uses over the C-ABI in ``include/rlra_c.h``.  It mirrors the
reference's C++ API names and semantics (``rlra::rsvd_v2``, ``qb_blocked``,
``id_rand``, ... in /root/reference/proj/include/rlra) so tests read like the
reference's own tests:

* matrices are numpy float64 arrays (any layout; converted to column-major);
* ``Rng`` is the reference's ``RngState`` (xoshiro256++/Box-Muller, consumed
  exactly as the reference consumes it when Omega comes from it);
* errors raise ``DimensionError`` / ``NumericalError`` / ``ConvergenceError``
  / ``IoError`` (all ``RlraError``), with the reference's message text.

Every call runs on the GPU through ``_lib/librlra_b200.so``; there is no CPU
fallback.  If the library or a CUDA device is missing the calls raise.

``Engine.device_*`` variants take raw device pointers (e.g. from
``torch.Tensor.data_ptr()``) and never touch host memory; bench.py uses them
for the device-resident timing.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "librlra_b200.so")
ROOT = os.path.dirname(_HERE)

HOST, DEVICE = 0, 1
RSVD_V2, RSVD_V1, RSVD_BASIC = 0, 1, 2
VNUM_QR, VNUM_BBT = 0, 1
OMEGA_CALLBACK, OMEGA_PHILOX = 0, 1

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i64 = C.c_int64


class RlraError(RuntimeError):
    """rlra::Error (reference core/errors.hpp:11-13)."""


class DimensionError(RlraError):
    """rlra::DimensionError (core/errors.hpp:16-18)."""


class NumericalError(RlraError):
    """rlra::NumericalError (core/errors.hpp:21-23)."""


class ConvergenceError(RlraError):
    """rlra::ConvergenceError (core/errors.hpp:26-28)."""


class IoError(RlraError):
    """rlra::IoError (core/errors.hpp:31-33)."""


_STATUS = {1: DimensionError, 2: NumericalError, 3: ConvergenceError, 4: IoError}


class _RngStruct(C.Structure):
    _fields_ = [("s", C.c_uint64 * 4), ("spare", C.c_double), ("have_spare", C.c_int)]


class _Omega(C.Structure):
    _fields_ = [("mode", C.c_int), ("fill", C.c_void_p), ("user", C.c_void_p),
                ("seed", C.c_uint64)]


class _RngNodes(C.Structure):  # rlra_rng_nodes
    _fields_ = [("nodes", C.c_void_p), ("count", C.c_int), ("substream_per_draw", C.c_int)]


_lib = None


def lib():
    """Load the engine library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RlraError(f"engine library missing: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        L.rlra_last_error.restype = C.c_char_p
        L.rlra_version.restype = C.c_char_p
        L.rlra_ctx_launch_count.restype = C.c_uint64
        L.rlra_ctx_launch_count.argtypes = [C.c_void_p]
        L.rlra_ctx_stream.restype = C.c_void_p
        L.rlra_ctx_stream.argtypes = [C.c_void_p]
        L.rlra_rng_next_u64.restype = C.c_uint64
        L.rlra_rng_next_gaussian.restype = C.c_double
        L.rlra_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.rlra_comm_destroy.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _check(st):
    if st != 0:
        msg = lib().rlra_last_error().decode()
        raise _STATUS.get(st, RlraError)(msg)


def _F(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _d(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _i(a):
    return a.ctypes.data_as(_ip) if a is not None else None


def _ld(a):
    return max(1, a.shape[0])


class Rng:
    """The reference's RngState (core/rng.hpp:18-79), host side."""

    def __init__(self, seed: int = 0):
        self._s = _RngStruct()
        lib().rlra_rng_seed(C.byref(self._s), C.c_uint64(seed))

    def next_u64(self) -> int:
        return int(lib().rlra_rng_next_u64(C.byref(self._s)))

    def next_gaussian(self) -> float:
        return float(lib().rlra_rng_next_gaussian(C.byref(self._s)))

    def substream(self) -> "Rng":
        child = Rng.__new__(Rng)
        child._s = _RngStruct()
        lib().rlra_rng_substream(C.byref(self._s), C.byref(child._s))
        return child

    def state(self):
        return (tuple(self._s.s), self._s.spare, self._s.have_spare)


def gaussian_matrix(rows: int, cols: int, rng: Rng) -> np.ndarray:
    """core/rng.hpp:82-87, column-major fill."""
    out = np.zeros((rows, cols), order="F")
    lib().rlra_rng_gaussian_fill(C.byref(rng._s), rows, cols, _d(out))
    return out


class Omega:
    """Gaussian test-matrix source for one call (rlra_omega in rlra_c.h).

    ``Omega.from_rng(rng)``      parity mode: the reference's stream, drawn on
                                 the host from ``rng`` in the reference's order.
    ``Omega.philox(seed)``       performance mode: Philox4x32-10 normals keyed
                                 by (seed, row, column, draw), materialised once
                                 per call (n x l) for the streaming GEMM, or
                                 generated in-register inside it with
                                 RLRA_SKETCH_FUSED=1 (same bits).
    """

    def __init__(self, mode, rng=None, seed=0, substream=False):
        self.mode = mode
        self.rng = rng
        self.seed = seed
        self.substream = substream

    @staticmethod
    def from_rng(rng: Rng, substream=False):
        return Omega(OMEGA_CALLBACK, rng=rng, substream=substream)

    @staticmethod
    def philox(seed: int):
        return Omega(OMEGA_PHILOX, seed=seed)

    def struct(self):
        L = lib()
        o = _Omega()
        o.mode = self.mode
        o.seed = self.seed
        if self.mode == OMEGA_CALLBACK:
            fn = L.rlra_omega_fill_rng_substream if self.substream else L.rlra_omega_fill_rng
            o.fill = C.cast(fn, C.c_void_p).value
            o.user = C.cast(C.pointer(self.rng._s), C.c_void_p).value
        return o


def _omega(omega, rng, substream=False):
    if omega is None:
        if rng is None:
            raise RlraError("need an Rng or an Omega")
        omega = Omega.from_rng(rng, substream)
    elif omega.mode == OMEGA_CALLBACK and substream:
        omega = Omega.from_rng(omega.rng, True)
    return omega


class _HostColl(C.Structure):  # rlra_host_collectives
    _fields_ = [("allreduce_sum", C.c_void_p), ("allgather", C.c_void_p), ("gpu_acquire", C.c_void_p),
                ("gpu_release", C.c_void_p), ("user", C.c_void_p)]


_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_size_t)
_ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_size_t)
_TOKEN_FN = C.CFUNCTYPE(None, C.c_void_p)


class HostCollectives:
    """Collectives written in Python for rlra_comm_create_host:
    ``allreduce_sum(buf)`` sums the float64 numpy array over the ranks in
    place; ``allgather(send, recv)`` fills recv[r*n:(r+1)*n] with rank r's
    send; ``gpu_acquire`` / ``gpu_release`` (optional) guard the GPU token.
    A Python exception fails the driver call with RLRA_ENCCL."""

    def __init__(self, allreduce_sum, allgather, gpu_acquire=None, gpu_release=None):
        import traceback

        def ar(_user, buf, count):
            try:
                allreduce_sum(np.ctypeslib.as_array(buf, (count,)))
                return 0
            except Exception:
                traceback.print_exc()
                return 1

        def ag(_user, send, recv, count):
            try:
                allgather(np.ctypeslib.as_array(send, (count,)),
                          np.ctypeslib.as_array(recv, (count * self.world_hint,)) if self.world_hint else None)
                return 0
            except Exception:
                traceback.print_exc()
                return 1

        self.world_hint = 0  # set by Engine.comm_create_host
        self._fns = [_ALLREDUCE_FN(ar), _ALLGATHER_FN(ag)]
        if (gpu_acquire is None) != (gpu_release is None):
            raise RlraError("gpu_acquire and gpu_release go together")
        if gpu_acquire is not None:
            self._fns += [_TOKEN_FN(lambda _u: gpu_acquire()), _TOKEN_FN(lambda _u: gpu_release())]

    def struct(self):
        h = _HostColl()
        h.allreduce_sum = C.cast(self._fns[0], C.c_void_p).value
        h.allgather = C.cast(self._fns[1], C.c_void_p).value
        if len(self._fns) == 4:
            h.gpu_acquire = C.cast(self._fns[2], C.c_void_p).value
            h.gpu_release = C.cast(self._fns[3], C.c_void_p).value
        return h


class LocalGroup:
    """rlra_local_group: ranks run as threads of this process (one Engine
    each), collectives over shared memory in C++ (sums in rank order on every
    rank), a barrier that fails after ``timeout_s`` instead of hanging, and a
    GPU token so ranks sharing one device take turns on it."""

    def __init__(self, nranks: int, timeout_s: float = 0.0):
        self._h = C.c_void_p()
        _check(lib().rlra_local_group_create(nranks, C.c_double(timeout_s), C.byref(self._h)))
        self.nranks = nranks

    def collectives(self, rank: int):
        h = _HostColl()
        _check(lib().rlra_local_group_collectives(self._h, rank, C.byref(h)))

        class _Fixed:
            world_hint = self.nranks

            @staticmethod
            def struct():
                return h

        return _Fixed()

    def close(self):
        if self._h:
            lib().rlra_local_group_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Engine:
    """One device context (rlra_ctx)."""

    def __init__(self, device: int = 0):
        L = lib()
        self._ctx = C.c_void_p()
        _check(L.rlra_ctx_create(device, C.byref(self._ctx)))
        self.device = device

    def close(self):
        if self._ctx:
            lib().rlra_ctx_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(lib().rlra_ctx_launch_count(self._ctx))

    @property
    def stream(self) -> int:
        return int(lib().rlra_ctx_stream(self._ctx) or 0)

    def synchronize(self):
        _check(lib().rlra_ctx_synchronize(self._ctx))

    # ------------------------------------------------------------ kernels --
    def matmul(self, a, b, trans_a=False, trans_b=False):
        a, b = _F(a), _F(b)
        m = a.shape[1] if trans_a else a.shape[0]
        n = b.shape[0] if trans_b else b.shape[1]
        c = np.zeros((m, n), order="F")
        _check(lib().rlra_matmul(self._ctx, HOST, int(trans_a), int(trans_b), _d(a), a.shape[0],
                                 a.shape[1], _i64(_ld(a)), _d(b), b.shape[0], b.shape[1],
                                 _i64(_ld(b)), _d(c), _i64(max(1, m))))
        return c

    def compact_qr(self, a):
        """Returns (q, r, degenerate_rank) — core/qr.hpp:95."""
        a = _F(a)
        m, n = a.shape
        q = np.zeros((m, n), order="F")
        r = np.zeros((n, n), order="F")
        deg = C.c_int(0)
        _check(lib().rlra_compact_qr(self._ctx, HOST, _d(a), m, n, _i64(_ld(a)), _d(q),
                                     _i64(max(1, m)), _d(r), _i64(max(1, n)), C.byref(deg)))
        return q, r, bool(deg.value)

    def orth(self, a):
        a = _F(a)
        m, n = a.shape
        q = np.zeros((m, n), order="F")
        deg = C.c_int(0)
        _check(lib().rlra_compact_qr(self._ctx, HOST, _d(a), m, n, _i64(_ld(a)), _d(q),
                                     _i64(max(1, m)), None, _i64(1), C.byref(deg)))
        return q

    def chol_inv(self, g, floor=0.0):
        """Upper Cholesky G = R^T R (upper triangle of g read) and R^{-1}:
        the CholQR kernel (qr.cu).  Returns (R, R^{-1}, ok)."""
        g = _F(g)
        n = g.shape[0]
        r = np.zeros((n, n), order="F")
        ri = np.zeros((n, n), order="F")
        ok = C.c_int(0)
        _check(lib().rlra_chol_inv(self._ctx, HOST, _d(g), n, _i64(_ld(g)), C.c_double(floor), _d(r),
                                   _i64(max(1, n)), _d(ri), _i64(max(1, n)), C.byref(ok)))
        return r, ri, bool(ok.value)

    def pivoted_qr_partial(self, a, k, tol=0.0):
        a = _F(a)
        m, n = a.shape
        kmax = min(m, n) if (k == 0 and tol > 0) else max(k, 1)
        q1 = np.zeros((m, kmax), order="F")
        s1 = np.zeros((kmax, n), order="F")
        perm = np.zeros(n, dtype=np.int32)
        frank, reached, deg = C.c_int(0), C.c_int(0), C.c_int(0)
        res = C.c_double(0)
        _check(lib().rlra_pivoted_qr(self._ctx, HOST, _d(a), m, n, _i64(_ld(a)), k,
                                     C.c_double(tol), _d(q1), _i64(max(1, m)), _d(s1),
                                     _i64(kmax), _i(perm), C.byref(frank), C.byref(res),
                                     C.byref(reached), C.byref(deg)))
        f = frank.value
        return dict(q1=q1[:, :f], s1=s1[:f], perm=perm, frank=f, residual=res.value,
                    tolerance_reached=bool(reached.value), degenerate_rank=bool(deg.value))

    def upper_tri_solve(self, s11, s12):
        s11, s12 = _F(s11), _F(s12)
        k, nc = s12.shape
        if s11.shape[0] != s11.shape[1]:
            raise DimensionError(f"upper_tri_solve: S11 is {s11.shape[0]}x{s11.shape[1]}, need square")
        if s11.shape[0] != k:
            raise DimensionError(f"upper_tri_solve: S12 has {k} rows, need {s11.shape[0]}")
        t = np.zeros((k, nc), order="F")
        cl = C.c_int(0)
        _check(lib().rlra_upper_tri_solve(self._ctx, HOST, _d(s11), k, _i64(_ld(s11)), _d(s12),
                                          nc, _i64(_ld(s12)), _d(t), _i64(max(1, k)),
                                          C.byref(cl)))
        return t, bool(cl.value)

    def small_svd(self, a):
        """Returns (u, sigma, v) — core/jacobi.hpp:145."""
        a = _F(a)
        m, n = a.shape
        r = min(m, n)
        u = np.zeros((m, r), order="F")
        s = np.zeros(r)
        v = np.zeros((n, r), order="F")
        _check(lib().rlra_small_svd(self._ctx, HOST, _d(a), m, n, _i64(_ld(a)), _d(u),
                                    _i64(max(1, m)), _d(s), _d(v), _i64(max(1, n))))
        return u, s, v

    def sym_eig(self, t):
        t = _F(t)
        n = t.shape[0]
        if t.shape[1] != n:
            raise DimensionError(f"sym_eig: matrix is {t.shape[0]}x{t.shape[1]}, need square")
        vals = np.zeros(n)
        vecs = np.zeros((n, n), order="F")
        _check(lib().rlra_sym_eig(self._ctx, HOST, _d(t), n, _i64(_ld(t)), _d(vals), _d(vecs),
                                  _i64(max(1, n))))
        return vals, vecs

    def frobenius_norm(self, a):
        a = _F(a)
        out = C.c_double(0)
        _check(lib().rlra_frobenius_norm(self._ctx, HOST, _d(a), a.shape[0], a.shape[1],
                                         _i64(_ld(a)), C.byref(out)))
        return out.value

    def gaussian_philox(self, rows, cols, seed, draw=0, row0=0):
        out = np.zeros((rows, cols), order="F")
        _check(lib().rlra_gaussian_philox(self._ctx, HOST, rows, cols, C.c_uint64(seed), draw,
                                          _i64(row0), _d(out), _i64(max(1, rows))))
        return out

    # --------------------------------------------------------- algorithms --
    def sample_right(self, a, l, q, s, rng=None, omega=None):
        return self._sample(a, l, q, s, rng, omega, left=False)

    def sample_left(self, a, l, q, s, rng=None, omega=None):
        return self._sample(a, l, q, s, rng, omega, left=True)

    def _sample(self, a, l, q, s, rng, omega, left):
        a = _F(a)
        m, n = a.shape
        om = _omega(omega, rng).struct()
        y = np.zeros((l, n) if left else (m, l), order="F")
        _check(lib().rlra_sample(self._ctx, HOST, int(left), _d(a), m, n, _i64(_ld(a)), l, q, s,
                                 C.byref(om), _d(y), _i64(max(1, y.shape[0]))))
        return y

    def _rsvd(self, variant, a, k, p, q, s, rng, omega):
        a = _F(a)
        m, n = a.shape
        om = _omega(omega, rng).struct()
        kk = max(k, 0)
        u = np.zeros((m, kk), order="F")
        sg = np.zeros(kk)
        v = np.zeros((n, kk), order="F")
        _check(lib().rlra_rsvd(self._ctx, HOST, variant, _d(a), m, n, _i64(_ld(a)), k, p, q, s,
                               C.byref(om), _d(u), _i64(max(1, m)), _d(sg), _d(v),
                               _i64(max(1, n))))
        return u, sg, v

    def rsvd_v2(self, a, k, p, q_power, s, rng=None, omega=None):
        """rsvd.hpp:154 — returns (u, sigma, v)."""
        return self._rsvd(RSVD_V2, a, k, p, q_power, s, rng, omega)

    def rsvd_v1(self, a, k, p, q_power, s, rng=None, omega=None):
        """rsvd.hpp:144."""
        return self._rsvd(RSVD_V1, a, k, p, q_power, s, rng, omega)

    def rsvd_basic(self, a, k, p, rng=None, omega=None):
        """rsvd.hpp:127."""
        return self._rsvd(RSVD_BASIC, a, k, p, 0, 1, rng, omega)

    def qb_blocked(self, a, b, num_blocks, tol, q_power, reorth_period, rng=None, omega=None,
                   inplace=False):
        """qb.hpp:148 (qb_blocked) / :98 (inplace: `a` must be a writable
        Fortran-ordered float64 array; it is left as A - QB)."""
        if inplace:
            if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.f_contiguous
                    and a.flags.writeable):
                raise RlraError("inplace qb_blocked needs a writable Fortran float64 array")
            A = a
        else:
            A = _F(a)
        m, n = A.shape
        cap = max(1, min(b * num_blocks, min(m, n))) if b >= 1 and num_blocks >= 1 else 1
        om = _omega(omega, rng, substream=True).struct()
        Q = np.zeros((m, cap), order="F")
        B = np.zeros((cap, n), order="F")
        hist = np.zeros(max(num_blocks, 1))
        ell, nh, reached = C.c_int(0), C.c_int(0), C.c_int(0)
        fin = C.c_double(0)
        _check(lib().rlra_qb_blocked(self._ctx, HOST, _d(A), m, n, _i64(_ld(A)), int(inplace), b,
                                     num_blocks, C.c_double(tol), q_power, reorth_period,
                                     C.byref(om), _d(Q), _i64(max(1, m)), _d(B), _i64(cap), cap,
                                     C.byref(ell), _d(hist), C.byref(nh), C.byref(fin),
                                     C.byref(reached)))
        e = ell.value
        return dict(q=np.asfortranarray(Q[:, :e]), b=np.asfortranarray(B[:e]), ell=e,
                    history=hist[:nh.value].copy(), final_residual=fin.value,
                    tolerance_reached=bool(reached.value))

    @staticmethod
    def _node_streams(rng, count, substream_per_draw):
        """rlra_rng_nodes of `count` substreams of rng, in the reference's order."""
        nodes = (_RngStruct * count)()
        for i in range(count):
            lib().rlra_rng_substream(C.byref(rng._s), C.byref(nodes[i]))
        holder = _RngNodes(C.cast(nodes, C.c_void_p), count, int(substream_per_draw))
        return nodes, holder

    def _composite_qb(self, fn, a, args, rank, rng, count, substream_per_draw):
        A = _F(a)
        m, n = A.shape
        nodes, holder = self._node_streams(rng, count, substream_per_draw)
        om = _Omega(OMEGA_CALLBACK, C.cast(lib().rlra_omega_fill_rng_nodes, C.c_void_p),
                          C.cast(C.pointer(holder), C.c_void_p), 0)
        Q = np.zeros((m, rank), order="F")
        B = np.zeros((rank, n), order="F")
        fin = C.c_double(0)
        _check(fn(self._ctx, HOST, _d(A), m, n, _i64(_ld(A)), *args, C.byref(om), _d(Q), _i64(max(1, m)), _d(B),
                  _i64(max(1, rank)), C.byref(fin)))
        return dict(q=Q, b=B, ell=rank, final_residual=fin.value, history=[fin.value], tolerance_reached=True)

    def qb_parallel(self, a, b, num_blocks, q_power, rng):
        """qb.hpp:159 (reference Omega streams: one substream per block)."""
        return self._composite_qb(lib().rlra_qb_parallel, a, (b, num_blocks, q_power), b * num_blocks, rng,
                                  num_blocks, False)

    def qb_hierarchical(self, a, num_row_blocks, b, num_blocks, q_power, rng):
        """qb.hpp:211 (reference streams: leaf substreams, then merge substreams)."""
        return self._composite_qb(lib().rlra_qb_hierarchical, a, (num_row_blocks, b, num_blocks, q_power),
                                  b * num_blocks, rng, 2 * num_row_blocks - 1, True)

    def qb_hierarchical_rowsharded(self, comm, a_local, m_total, num_row_blocks, b, num_blocks, q_power, rng):
        """rlra_qb_hierarchical_rowsharded with host buffers (this rank's slabs)."""
        fn = lib().rlra_qb_hierarchical_rowsharded
        A = _F(a_local)
        mg, n = A.shape
        rank = b * num_blocks
        nodes, holder = self._node_streams(rng, 2 * num_row_blocks - 1, True)
        om = _Omega(OMEGA_CALLBACK, C.cast(lib().rlra_omega_fill_rng_nodes, C.c_void_p),
                    C.cast(C.pointer(holder), C.c_void_p), 0)
        Q = np.zeros((mg, rank), order="F")
        B = np.zeros((rank, n), order="F")
        fin = C.c_double(0)
        _check(fn(self._ctx, comm, HOST, _d(A), mg, n, _i64(_ld(A)), _i64(m_total), num_row_blocks, b, num_blocks,
                  q_power, C.byref(om), _d(Q), _i64(max(1, mg)), _d(B), _i64(max(1, rank)), C.byref(fin)))
        return dict(q=Q, b=B, ell=rank, final_residual=fin.value)

    def svd_from_qb(self, qb, k=0, vnum=VNUM_QR):
        """qb.hpp:276 — qb is the dict qb_blocked returns."""
        q, b = _F(qb["q"]), _F(qb["b"])
        m, ell = q.shape
        n = b.shape[1]
        kk = ell if k == 0 else k
        u = np.zeros((m, max(kk, 0)), order="F")
        s = np.zeros(max(kk, 0))
        v = np.zeros((n, max(kk, 0)), order="F")
        ko = C.c_int(0)
        _check(lib().rlra_svd_from_qb(self._ctx, HOST, _d(q), m, _i64(max(1, m)), _d(b), n,
                                      _i64(max(1, ell)), ell, k, vnum, _d(u) if kk > 0 else None,
                                      _i64(max(1, m)), _d(s) if kk > 0 else None,
                                      _d(v) if kk > 0 else None, _i64(max(1, n)), C.byref(ko)))
        kk = ko.value
        return u[:, :kk], s[:kk], v[:, :kk]

    def id_column(self, a, k, tol=0.0):
        """interp.hpp:101 — returns dict(jc, v, k, qr_residual, tolerance_reached, clamped)."""
        a = _F(a)
        m, n = a.shape
        kcap = min(m, n) if (k == 0 and tol > 0) else max(k, 1)
        jc = np.zeros(n, dtype=np.int32)
        v = np.zeros((n, kcap), order="F")
        ko, reached, cl = C.c_int(0), C.c_int(0), C.c_int(0)
        res = C.c_double(0)
        _check(lib().rlra_id_column(self._ctx, HOST, _d(a), m, n, _i64(_ld(a)), k,
                                    C.c_double(tol), _i(jc), _d(v), _i64(max(1, n)), C.byref(ko),
                                    C.byref(res), C.byref(reached), C.byref(cl)))
        kk = ko.value
        return dict(jc=jc, v=np.asfortranarray(v[:, :kk]), k=kk, qr_residual=res.value,
                    tolerance_reached=bool(reached.value), clamped=bool(cl.value))

    def id_row(self, a, k, tol=0.0):
        """interp.hpp:107 — column ID of A^T with the roles renamed."""
        r = self.id_column(np.asarray(a, dtype=np.float64).T, k, tol)
        return dict(jr=r["jc"], w=r["v"], k=r["k"], qr_residual=r["qr_residual"],
                    tolerance_reached=r["tolerance_reached"], clamped=r["clamped"])

    def id_rand(self, a, k, p, q_power, s, rng=None, omega=None):
        """interp.hpp:203."""
        a = _F(a)
        m, n = a.shape
        om = _omega(omega, rng).struct()
        jc = np.zeros(n, dtype=np.int32)
        v = np.zeros((n, max(k, 0)), order="F")
        res, cl = C.c_double(0), C.c_int(0)
        _check(lib().rlra_id_rand(self._ctx, HOST, _d(a), m, n, _i64(_ld(a)), k, p, q_power, s,
                                  C.byref(om), _i(jc), _d(v), _i64(max(1, n)), C.byref(res),
                                  C.byref(cl)))
        return dict(jc=jc, v=v, k=k, qr_residual=res.value, tolerance_reached=True,
                    clamped=bool(cl.value))

    def two_sided_from_column(self, a, col):
        """interp.hpp:123 — col is an id dict; returns a two-sided dict."""
        a = _F(a)
        m, n = a.shape
        k = col["k"]
        jc = np.ascontiguousarray(col["jc"], dtype=np.int32)
        jr = np.zeros(m, dtype=np.int32)
        w = np.zeros((m, max(k, 0)), order="F")
        _check(lib().rlra_two_sided_from_column(self._ctx, HOST, _d(a), m, n, _i64(_ld(a)),
                                                _i(jc), k, _i(jr), _d(w) if k > 0 else None,
                                                _i64(max(1, m))))
        return dict(jr=jr, jc=jc, w=w, v=col["v"], k=k, qr_residual=col["qr_residual"],
                    tolerance_reached=col.get("tolerance_reached", True))

    def id_two_sided(self, a, k, tol=0.0):
        """interp.hpp:190."""
        return self.two_sided_from_column(a, self.id_column(a, k, tol))

    def cur_from_two_sided(self, a, ts):
        """interp.hpp:158."""
        a = _F(a)
        m, n = a.shape
        k = ts["k"]
        jc = np.ascontiguousarray(ts["jc"], dtype=np.int32)
        jr = np.ascontiguousarray(ts["jr"], dtype=np.int32)
        v = _F(ts["v"]) if k > 0 else np.zeros((n, 1), order="F")
        c = np.zeros((m, k), order="F")
        u = np.zeros((k, k), order="F")
        r = np.zeros((k, n), order="F")
        res = C.c_double(0)
        _check(lib().rlra_cur_from_two_sided(self._ctx, HOST, _d(a), m, n, _i64(_ld(a)), _i(jc),
                                             _i(jr), _d(v), _i64(max(1, n)), k,
                                             _d(c) if k else None, _i64(max(1, m)),
                                             _d(u) if k else None, _i64(max(1, k)),
                                             _d(r) if k else None, _i64(max(1, k)),
                                             C.byref(res)))
        return dict(c=c, u=u, r=r, jr=jr, jc=jc, k=k, residual=res.value,
                    qr_residual=ts["qr_residual"], tolerance_reached=ts.get("tolerance_reached", True))

    def cur(self, a, k, tol=0.0):
        """interp.hpp:196."""
        return self.cur_from_two_sided(a, self.id_two_sided(a, k, tol))

    def cur_rand(self, a, k, p, q_power, s, rng=None, omega=None):
        """interp.hpp:240."""
        a = _F(a)
        m, n = a.shape
        om = _omega(omega, rng).struct()
        jc = np.zeros(n, dtype=np.int32)
        jr = np.zeros(m, dtype=np.int32)
        v = np.zeros((n, k), order="F")
        w = np.zeros((m, k), order="F")
        c = np.zeros((m, k), order="F")
        u = np.zeros((k, k), order="F")
        r = np.zeros((k, n), order="F")
        res, qres = C.c_double(0), C.c_double(0)
        _check(lib().rlra_cur_rand(self._ctx, HOST, _d(a), m, n, _i64(_ld(a)), k, p, q_power, s,
                                   C.byref(om), _i(jc), _i(jr), _d(v), _i64(max(1, n)), _d(w),
                                   _i64(max(1, m)), _d(c), _i64(max(1, m)), _d(u),
                                   _i64(max(1, k)), _d(r), _i64(max(1, k)), C.byref(res),
                                   C.byref(qres)))
        return dict(c=c, u=u, r=r, jr=jr, jc=jc, v=v, w=w, k=k, residual=res.value,
                    qr_residual=qres.value, tolerance_reached=True)

    def id_from_qb(self, qb, a, k):
        """interp.hpp:228."""
        a = np.asarray(a)
        if a.shape[0] != qb["q"].shape[0] or a.shape[1] != qb["b"].shape[1]:
            raise DimensionError(
                f"id_from_qb: matrix is {a.shape[0]}x{a.shape[1]} but the QB factors describe "
                f"{qb['q'].shape[0]}x{qb['b'].shape[1]}")
        if k < 1 or k > qb["ell"]:
            raise DimensionError(f"rank k = {k} outside [1, rank(B) = {qb['ell']}]")
        return self.id_column(qb["b"], k, 0.0)

    # ------------------------------------------------- device-pointer API --
    def device_rsvd(self, variant, a_ptr, m, n, lda, k, p, q, s, omega, u_ptr, sigma_ptr, v_ptr):
        om = omega.struct()
        _check(lib().rlra_rsvd(self._ctx, DEVICE, variant, C.c_void_p(a_ptr), m, n, _i64(lda), k,
                               p, q, s, C.byref(om), C.c_void_p(u_ptr), _i64(m),
                               C.c_void_p(sigma_ptr), C.c_void_p(v_ptr), _i64(n)))

    # -- row-sharded multi-GPU path (C++ driver + NCCL, csrc/dist.cu) ----------
    @staticmethod
    def comm_unique_id() -> bytes:
        """rlra_comm_unique_id: the 128-byte NCCL id rank 0 distributes."""
        buf = (C.c_ubyte * 128)()
        _check(lib().rlra_comm_unique_id(buf))
        return bytes(buf)

    def comm_create(self, uid: bytes, nranks: int, rank: int):
        if len(uid) != 128:
            raise RlraError("NCCL unique id must be 128 bytes")
        h = C.c_void_p()
        _check(lib().rlra_comm_create(self._ctx, (C.c_ubyte * 128).from_buffer_copy(uid), nranks, rank,
                                      C.byref(h)))
        return h

    def comm_create_host(self, nranks: int, rank: int, collectives):
        """rlra_comm_create_host over HostCollectives (Python) or
        LocalGroup.collectives(rank) (C++ shared memory)."""
        if isinstance(collectives, HostCollectives):
            collectives.world_hint = nranks
        h = C.c_void_p()
        hc = collectives.struct()
        self._keep_coll = getattr(self, "_keep_coll", []) + [collectives, hc]
        _check(lib().rlra_comm_create_host(self._ctx, nranks, rank, C.byref(hc), C.byref(h)))
        return h

    def device_gen_test_matrix_rowsharded(self, comm, row0, m_local, m_total, n, sigma, seed, noise, out_ptr, ld):
        sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        _check(lib().rlra_gen_test_matrix_rowsharded(self._ctx, comm, DEVICE, _i64(row0), m_local, _i64(m_total), n,
                                                     _d(sigma), len(sigma), C.c_uint64(seed), C.c_double(noise),
                                                     C.c_void_p(out_ptr), _i64(ld)))

    def rsvd_rowsharded(self, comm, a_local, m_total, k, p, q, s, rng=None, omega=None):
        """rlra_rsvd_rowsharded with host buffers: (U_g, sigma, V)."""
        a = _F(a_local)
        mg, n = a.shape
        om = _omega(omega, rng).struct()
        u = np.zeros((mg, k), order="F")
        sg = np.zeros(k)
        v = np.zeros((n, k), order="F")
        _check(lib().rlra_rsvd_rowsharded(self._ctx, comm, HOST, _d(a), mg, n, _i64(_ld(a)), _i64(m_total), k, p,
                                          q, s, C.byref(om), _d(u), _i64(max(1, mg)), _d(sg), _d(v),
                                          _i64(max(1, n))))
        return u, sg, v

    @staticmethod
    def comm_destroy(h):
        lib().rlra_comm_destroy(h)

    def device_rsvd_rowsharded(self, comm, a_ptr, m_local, n, lda, m_total, k, p, q, s, omega, u_ptr, ldu,
                               sigma_ptr, v_ptr, ldv, loc=None):
        om = omega.struct()
        _check(lib().rlra_rsvd_rowsharded(self._ctx, comm, DEVICE if loc is None else loc, C.c_void_p(a_ptr),
                                          m_local, n, _i64(lda), _i64(m_total), k, p, q, s, C.byref(om),
                                          C.c_void_p(u_ptr), _i64(ldu), C.c_void_p(sigma_ptr), C.c_void_p(v_ptr),
                                          _i64(ldv)))

    def host_rsvd_rowsharded_ptr(self, comm, a_ptr, m_local, n, lda, m_total, k, p, q, s, omega, u_ptr, ldu,
                                 sigma_ptr, v_ptr, ldv):
        """rlra_rsvd_rowsharded with this rank's shard in HOST memory: the
        upload streams in row chunks under the local sketch GEMM."""
        self.device_rsvd_rowsharded(comm, a_ptr, m_local, n, lda, m_total, k, p, q, s, omega, u_ptr, ldu,
                                    sigma_ptr, v_ptr, ldv, loc=HOST)

    def id_rand_rowsharded(self, comm, a_local, row0, m_total, k, p, q_power, s, rng=None, omega=None):
        """rlra_id_rand_rowsharded with host buffers: a_local is this rank's
        rows [row0, row0 + m_local) of A."""
        a = _F(a_local)
        mg, n = a.shape
        om = _omega(omega, rng).struct()
        jc = np.zeros(n, dtype=np.int32)
        v = np.zeros((n, k), order="F")
        res, cl = C.c_double(0), C.c_int(0)
        _check(lib().rlra_id_rand_rowsharded(self._ctx, comm, HOST, _d(a), mg, n, _i64(_ld(a)), _i64(row0),
                                             _i64(m_total), k, p, q_power, s, C.byref(om), _i(jc), _d(v),
                                             _i64(max(1, n)), C.byref(res), C.byref(cl)))
        return dict(jc=jc, v=v, k=k, qr_residual=res.value, clamped=bool(cl.value))

    def qb_blocked_rowsharded(self, comm, a_local, m_total, b, num_blocks, tol, q_power, reorth_period,
                              rng=None, omega=None):
        """rlra_qb_blocked_rowsharded with host buffers: Q rows of this rank,
        B replicated."""
        a = _F(a_local)
        mg, n = a.shape
        om = _omega(omega, rng, substream=True).struct()
        cap = int(min(b * num_blocks, min(m_total, n)))
        q = np.zeros((mg, max(cap, 1)), order="F")
        bb = np.zeros((max(cap, 1), n), order="F")
        hist = np.zeros(max(num_blocks, 1))
        ell, nh, reached = C.c_int(0), C.c_int(0), C.c_int(0)
        fin = C.c_double(0)
        _check(lib().rlra_qb_blocked_rowsharded(self._ctx, comm, HOST, _d(a), mg, n, _i64(_ld(a)), _i64(m_total), 0,
                                                b, num_blocks, C.c_double(tol), q_power, reorth_period,
                                                C.byref(om), _d(q), _i64(max(1, mg)), _d(bb), _i64(max(cap, 1)), cap,
                                                C.byref(ell), _d(hist), C.byref(nh), C.byref(fin), C.byref(reached)))
        e = ell.value
        return dict(q=q[:, :e], b=bb[:e], ell=e, history=list(hist[: nh.value]), final_residual=fin.value,
                    tolerance_reached=bool(reached.value))

    def cur_rand_rowsharded(self, comm, a_local, row0, m_total, k, p, q_power, s, rng=None, omega=None):
        """rlra_cur_rand_rowsharded with host buffers (this rank's rows)."""
        a = _F(a_local)
        mg, n = a.shape
        om = _omega(omega, rng).struct()
        jc = np.zeros(n, dtype=np.int32)
        jr = np.zeros(k, dtype=np.int32)
        v = np.zeros((n, k), order="F")
        w = np.zeros((mg, k), order="F")
        c = np.zeros((mg, k), order="F")
        u = np.zeros((k, k), order="F")
        r = np.zeros((k, n), order="F")
        res, qres = C.c_double(0), C.c_double(0)
        _check(lib().rlra_cur_rand_rowsharded(self._ctx, comm, HOST, _d(a), mg, n, _i64(_ld(a)), _i64(row0),
                                              _i64(m_total), k, p, q_power, s, C.byref(om), _i(jc), _i(jr),
                                              _d(v), _i64(max(1, n)), _d(w), _i64(max(1, mg)), _d(c),
                                              _i64(max(1, mg)), _d(u), _i64(max(1, k)), _d(r), _i64(max(1, k)),
                                              C.byref(res), C.byref(qres)))
        return dict(jc=jc, jr=jr, v=v, w=w, c=c, u=u, r=r, k=k, residual=res.value, qr_residual=qres.value)

    # -- binary I/O, generator, verifier (csrc/io.cu) ---------------------------
    @staticmethod
    def binary_header(path):
        """(rows, cols) of a reference-format binary file (io.hpp:66-93 checks)."""
        r, c = C.c_int(0), C.c_int(0)
        _check(lib().rlra_binary_header(os.fsencode(path), C.byref(r), C.byref(c)))
        return r.value, c.value

    def load_binary(self, path, row0=0, rows=None):
        """Rows [row0, row0 + rows) of the file as a column-major array."""
        m, n = self.binary_header(path)
        rows = m - row0 if rows is None else rows
        out = np.zeros((rows, n), order="F")
        _check(lib().rlra_load_binary(self._ctx, HOST, os.fsencode(path), _i64(row0), rows, _d(out),
                                      _i64(max(1, rows))))
        return out

    def device_load_binary(self, path, row0, rows, out_ptr, ld):
        _check(lib().rlra_load_binary(self._ctx, DEVICE, os.fsencode(path), _i64(row0), rows,
                                      C.c_void_p(out_ptr), _i64(ld)))

    def save_binary(self, path, a):
        a = _F(a)
        m, n = a.shape
        _check(lib().rlra_save_binary(self._ctx, HOST, os.fsencode(path), _d(a), m, n, _i64(_ld(a))))

    def gen_test_matrix(self, m, n, sigma, seed, noise=0.0):
        sg = np.ascontiguousarray(sigma, dtype=np.float64)
        out = np.zeros((m, n), order="F")
        _check(lib().rlra_gen_test_matrix(self._ctx, HOST, m, n, _d(sg), len(sg), C.c_uint64(seed),
                                          C.c_double(noise), _d(out), _i64(max(1, m))))
        return out

    def device_gen_test_matrix(self, m, n, sigma, seed, noise, out_ptr, ld):
        sg = np.ascontiguousarray(sigma, dtype=np.float64)
        _check(lib().rlra_gen_test_matrix(self._ctx, DEVICE, m, n, _d(sg), len(sg), C.c_uint64(seed),
                                          C.c_double(noise), C.c_void_p(out_ptr), _i64(ld)))

    def verify_svd(self, a, u, s, v, sigma_true=None):
        """report.hpp verify(a, SvdFactors, sigma_true)."""
        a, u, v = _F(a), _F(u), _F(v)
        m, n = a.shape
        k = u.shape[1]
        s = np.ascontiguousarray(s, dtype=np.float64)
        st = np.ascontiguousarray(sigma_true if sigma_true is not None else np.zeros(0), dtype=np.float64)
        out = np.zeros(5)
        _check(lib().rlra_verify_svd(self._ctx, HOST, _d(a), m, n, _i64(_ld(a)), _d(u), _i64(max(1, m)), _d(s),
                                     _d(v), _i64(max(1, n)), k, _d(st) if len(st) else None, len(st), _d(out)))
        return dict(rel_frobenius_error=out[0], rel_spectral_error=out[1], fro_floor=out[2],
                    spec_floor=out[3], spec_bound=out[4])

    def host_rsvd_ptr(self, variant, a_ptr, m, n, lda, k, p, q, s, omega, u_ptr, sigma_ptr, v_ptr):
        """rlra_rsvd with HOST pointers (pinned or pageable): the drop-in call
        a reference user makes, H2D/D2H inside the call."""
        om = omega.struct()
        _check(lib().rlra_rsvd(self._ctx, HOST, variant, C.c_void_p(a_ptr), m, n, _i64(lda), k,
                               p, q, s, C.byref(om), C.c_void_p(u_ptr), _i64(m),
                               C.c_void_p(sigma_ptr), C.c_void_p(v_ptr), _i64(n)))

    def device_qb_blocked(self, a_ptr, m, n, lda, inplace, b, num_blocks, tol, q_power,
                          reorth_period, omega, q_ptr, ldq, b_ptr, ldb, cap):
        """rlra_qb_blocked on device buffers; omega in callback mode must use
        substreams (Omega.from_rng(rng, substream=True))."""
        om = omega.struct()
        hist = np.zeros(max(num_blocks, 1))
        ell, nh, reached = C.c_int(0), C.c_int(0), C.c_int(0)
        fin = C.c_double(0)
        _check(lib().rlra_qb_blocked(self._ctx, DEVICE, C.c_void_p(a_ptr), m, n, _i64(lda),
                                     int(inplace), b, num_blocks, C.c_double(tol), q_power,
                                     reorth_period, C.byref(om), C.c_void_p(q_ptr), _i64(ldq),
                                     C.c_void_p(b_ptr), _i64(ldb), cap, C.byref(ell), _d(hist),
                                     C.byref(nh), C.byref(fin), C.byref(reached)))
        return dict(ell=ell.value, history=hist[:nh.value].copy(), final_residual=fin.value,
                    tolerance_reached=bool(reached.value))

    def device_svd_from_qb(self, q_ptr, m, ldq, b_ptr, n, ldb, ell, k, vnum, u_ptr, ldu, s_ptr,
                           v_ptr, ldv):
        ko = C.c_int(0)
        _check(lib().rlra_svd_from_qb(self._ctx, DEVICE, C.c_void_p(q_ptr), m, _i64(ldq),
                                      C.c_void_p(b_ptr), n, _i64(ldb), ell, k, vnum,
                                      C.c_void_p(u_ptr), _i64(ldu), C.c_void_p(s_ptr),
                                      C.c_void_p(v_ptr), _i64(ldv), C.byref(ko)))
        return ko.value

    def device_cur_rand(self, a_ptr, m, n, lda, k, p, q, s, omega, out):
        """rlra_cur_rand on device buffers; `out` maps jc, jr, v, w, c, u, r to
        device pointers (int32 / float64, leading dimensions n, m, m, k, k).
        Returns (residual, qr_residual)."""
        om = omega.struct()
        res, qres = C.c_double(0), C.c_double(0)
        _check(lib().rlra_cur_rand(self._ctx, DEVICE, C.c_void_p(a_ptr), m, n, _i64(lda), k, p, q, s, C.byref(om),
                                   C.c_void_p(out["jc"]), C.c_void_p(out["jr"]), C.c_void_p(out["v"]),
                                   _i64(max(1, n)), C.c_void_p(out["w"]), _i64(max(1, m)), C.c_void_p(out["c"]),
                                   _i64(max(1, m)), C.c_void_p(out["u"]), _i64(max(1, k)), C.c_void_p(out["r"]),
                                   _i64(max(1, k)), C.byref(res), C.byref(qres)))
        return res.value, qres.value

    def device_id_rand(self, a_ptr, m, n, lda, k, p, q, s, omega, jc_ptr, v_ptr, ldv):
        om = omega.struct()
        res, cl = C.c_double(0), C.c_int(0)
        _check(lib().rlra_id_rand(self._ctx, DEVICE, C.c_void_p(a_ptr), m, n, _i64(lda), k, p, q,
                                  s, C.byref(om), C.c_void_p(jc_ptr), C.c_void_p(v_ptr),
                                  _i64(ldv), C.byref(res), C.byref(cl)))
        return dict(qr_residual=res.value, clamped=bool(cl.value))

    # -- row-sharded building blocks (dist.py) --------------------------------
    def device_sketch(self, trans, a_ptr, m, n, lda, l, omega, draw, row0, y_ptr, ldy):
        om = omega.struct()
        _check(lib().rlra_sketch(self._ctx, DEVICE, int(trans), C.c_void_p(a_ptr), m, n, _i64(lda),
                                 l, C.byref(om), draw, _i64(row0), C.c_void_p(y_ptr), _i64(ldy)))

    def device_gram(self, y_ptr, m, n, ldy, g_ptr, ldg):
        _check(lib().rlra_gram(self._ctx, DEVICE, C.c_void_p(y_ptr), m, n, _i64(ldy),
                               C.c_void_p(g_ptr), _i64(ldg)))

    def device_chol_inv(self, g_ptr, n, ldg, floor, r_ptr, ldr, ri_ptr, ldri):
        ok = C.c_int(0)
        _check(lib().rlra_chol_inv(self._ctx, DEVICE, C.c_void_p(g_ptr), n, _i64(ldg),
                                   C.c_double(floor), C.c_void_p(r_ptr), _i64(ldr),
                                   C.c_void_p(ri_ptr), _i64(ldri), C.byref(ok)))
        return bool(ok.value)

    def device_trmm_right_upper(self, y_ptr, m, n, ldy, t_ptr, ldt, o_ptr, ldo):
        _check(lib().rlra_trmm_right_upper(self._ctx, DEVICE, C.c_void_p(y_ptr), m, n, _i64(ldy),
                                           C.c_void_p(t_ptr), _i64(ldt), C.c_void_p(o_ptr),
                                           _i64(ldo)))

    def device_compact_qr(self, a_ptr, m, n, lda, q_ptr, ldq, r_ptr, ldr):
        deg = C.c_int(0)
        _check(lib().rlra_compact_qr(self._ctx, DEVICE, C.c_void_p(a_ptr), m, n, _i64(lda),
                                     C.c_void_p(q_ptr), _i64(ldq),
                                     C.c_void_p(r_ptr) if r_ptr else None, _i64(ldr),
                                     C.byref(deg)))
        return bool(deg.value)

    def device_small_svd(self, a_ptr, m, n, lda, u_ptr, ldu, s_ptr, v_ptr, ldv):
        _check(lib().rlra_small_svd(self._ctx, DEVICE, C.c_void_p(a_ptr), m, n, _i64(lda),
                                    C.c_void_p(u_ptr), _i64(ldu), C.c_void_p(s_ptr),
                                    C.c_void_p(v_ptr), _i64(ldv)))

    def device_matmul(self, ta, tb, a_ptr, ar, ac, lda, b_ptr, br, bc, ldb, c_ptr, ldc):
        _check(lib().rlra_matmul(self._ctx, DEVICE, int(ta), int(tb), C.c_void_p(a_ptr), ar, ac,
                                 _i64(lda), C.c_void_p(b_ptr), br, bc, _i64(ldb),
                                 C.c_void_p(c_ptr), _i64(ldc)))

    def device_orth(self, a_ptr, m, n, lda=None):
        """In-place orthonormalisation of a device m x n matrix (CholQR2)."""
        lda = lda or m
        _check(lib().rlra_compact_qr(self._ctx, DEVICE, C.c_void_p(a_ptr), m, n, _i64(lda),
                                     C.c_void_p(a_ptr), _i64(lda), None, _i64(1), None))

    def device_lowrank_residual(self, a_ptr, m, n, lda, x_ptr, ldx, y_ptr, ldy, k):
        out = C.c_double(0)
        _check(lib().rlra_lowrank_residual(self._ctx, DEVICE, C.c_void_p(a_ptr), m, n, _i64(lda),
                                           C.c_void_p(x_ptr), _i64(ldx), C.c_void_p(y_ptr),
                                           _i64(ldy), k, C.byref(out)))
        return out.value

    def lowrank_residual(self, a, x, y):
        a, x, y = _F(a), _F(x), _F(y)
        out = C.c_double(0)
        _check(lib().rlra_lowrank_residual(self._ctx, HOST, _d(a), a.shape[0], a.shape[1],
                                           _i64(_ld(a)), _d(x), _i64(_ld(x)), _d(y), _i64(_ld(y)),
                                           x.shape[1], C.byref(out)))
        return out.value

    def device_rel_error(self, a_ptr, m, n, u_ptr, s_ptr, v_ptr, k):
        """||A - U diag(s) V^T||_F / ||A||_F for device factors (torch-free)."""
        import torch  # only for the scaled copy of U
        U = torch.empty(m * k, dtype=torch.float64, device=f"cuda:{self.device}")
        U.copy_(_wrap_dev(u_ptr, m * k, self.device))
        S = _wrap_dev(s_ptr, k, self.device)
        U.view(k, m).mul_(S.view(k, 1))
        torch.cuda.synchronize(self.device)
        r = self.device_lowrank_residual(a_ptr, m, n, m, U.data_ptr(), m, v_ptr, n, k)
        an = C.c_double(0)
        _check(lib().rlra_frobenius_norm(self._ctx, DEVICE, C.c_void_p(a_ptr), m, n, _i64(m),
                                         C.byref(an)))
        return r / an.value if an.value > 0 else r

    def profile(self, enable=True):
        _check(lib().rlra_ctx_profile(self._ctx, int(enable)))

    def profile_records(self):
        L = lib()
        out = []
        name = C.create_string_buffer(64)
        for i in range(L.rlra_ctx_profile_count(self._ctx)):
            M, N, K = C.c_int(0), C.c_int(0), C.c_int(0)
            fl, ms = C.c_double(0), C.c_double(0)
            _check(L.rlra_ctx_profile_get(self._ctx, i, name, 64, C.byref(M), C.byref(N),
                                          C.byref(K), C.byref(fl), C.byref(ms)))
            out.append(dict(name=name.value.decode(), M=M.value, N=N.value, K=K.value,
                            flops=fl.value, ms=ms.value))
        return out

    def device_gaussian_philox(self, rows, cols, seed, draw, row0, out_ptr, ld):
        _check(lib().rlra_gaussian_philox(self._ctx, DEVICE, rows, cols, C.c_uint64(seed), draw,
                                          _i64(row0), C.c_void_p(out_ptr), _i64(ld)))


def _wrap_dev(ptr, count, device):
    """A torch view of `count` device doubles at `ptr` (no copy)."""
    import torch

    class _CAI:
        __cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_CAI(), device=f"cuda:{device}")


_default = None


def default_engine() -> Engine:
    global _default
    if _default is None:
        _default = Engine(0)
    return _default
