"""ctypes front for the CPU parity checker (oracle/) — TEST INFRASTRUCTURE.

Two libraries with the same signatures:
  * ``orc``  — oracle/_build/librlra_oracle.so, our C restatement;
  * ``ref``  — oracle/_ref/librlra_ref.so, the unmodified reference headers
    behind a C-ABI shim (present where /root/reference was, or where the built
    file travelled with the repo snapshot).

Both take column-major float64 arrays (numpy ``order='F'``).  This module is
imported only by tests/, __graft_entry__.smoke() and bench.py's CPU legs.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORC_PATH = os.path.join(ORACLE_DIR, "_build", "librlra_oracle.so")
REF_PATH = os.path.join(ORACLE_DIR, "_ref", "librlra_ref.so")
REF_FAST_PATH = os.path.join(ORACLE_DIR, "_ref", "librlra_ref_fast.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class Rng(C.Structure):
    _fields_ = [("s", C.c_uint64 * 4), ("spare", C.c_double), ("have_spare", C.c_int)]


def _ensure_built():
    if not os.path.exists(ORC_PATH):
        subprocess.run(["make", "-C", ORACLE_DIR, "all"], check=True, capture_output=True)


def d(a):
    return a.ctypes.data_as(_dp)


def i(a):
    return a.ctypes.data_as(_ip)


def F(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


class _Lib:
    """Thin typed wrapper; prefix is 'orc_' or 'ref_'."""

    def __init__(self, path, prefix):
        self.lib = C.CDLL(path)
        self.p = prefix
        self.path = path
        for name, res in [("last_error", C.c_char_p)]:
            getattr(self.lib, prefix + name).restype = res

    def f(self, name):
        fn = getattr(self.lib, self.p + name)
        return fn

    def _chk(self, st):
        if st != 0:
            raise OracleError(st, self.f("last_error")().decode())

    # --- rng -----------------------------------------------------------
    def rng(self, seed):
        r = Rng()
        self.f("rng_seed")(C.byref(r), C.c_uint64(seed))
        return r

    def gaussian(self, rows, cols, r):
        out = np.zeros((rows, cols), order="F")
        self.f("gaussian_matrix")(rows, cols, C.byref(r), d(out))
        return out

    def substream(self, r):
        c = Rng()
        self.f("rng_substream")(C.byref(r), C.byref(c))
        return c

    # --- kernels ----------------------------------------------------------
    def matmul(self, a, b, ta=False, tb=False):
        a, b = F(a), F(b)
        m = a.shape[1] if ta else a.shape[0]
        n = b.shape[0] if tb else b.shape[1]
        c = np.zeros((m, n), order="F")
        self._chk(self.f("matmul")(int(ta), int(tb), d(a), a.shape[0], a.shape[1], d(b),
                                   b.shape[0], b.shape[1], d(c)))
        return c

    def compact_qr(self, a):
        a = F(a)
        m, n = a.shape
        q = np.zeros((m, n), order="F")
        r = np.zeros((n, n), order="F")
        deg = C.c_int(0)
        self._chk(self.f("compact_qr")(d(a), m, n, d(q), d(r), C.byref(deg)))
        return q, r, bool(deg.value)

    def pivoted_qr(self, a, k, tol=0.0):
        a = F(a)
        m, n = a.shape
        kmax = min(m, n) if (k == 0 and tol > 0) else max(k, 1)
        q1 = np.zeros((m, kmax), order="F")
        s1 = np.zeros((kmax, n), order="F")
        perm = np.zeros(n, dtype=np.int32)
        frank, reached, deg = C.c_int(0), C.c_int(0), C.c_int(0)
        res = C.c_double(0)
        self._chk(self.f("pivoted_qr")(d(a), m, n, k, C.c_double(tol), d(q1), d(s1), kmax, i(perm),
                                       C.byref(frank), C.byref(res), C.byref(reached),
                                       C.byref(deg)))
        f = frank.value
        return dict(q1=q1[:, :f].copy(order="F"), s1=s1[:f].copy(order="F"), perm=perm,
                    frank=f, residual=res.value, reached=bool(reached.value),
                    degenerate=bool(deg.value))

    def upper_tri_solve(self, s11, s12):
        s11, s12 = F(s11), F(s12)
        k, nc = s12.shape
        t = np.zeros((k, nc), order="F")
        cl = C.c_int(0)
        if self.p == "orc_":
            st = self.f("upper_tri_solve")(d(s11), k, k, d(s12), k, nc, d(t), C.byref(cl))
        else:
            st = self.f("upper_tri_solve")(d(s11), k, d(s12), nc, d(t), C.byref(cl))
        self._chk(st)
        return t, bool(cl.value)

    def small_svd(self, a):
        a = F(a)
        m, n = a.shape
        r = min(m, n)
        u = np.zeros((m, r), order="F")
        s = np.zeros(r)
        v = np.zeros((n, r), order="F")
        self._chk(self.f("small_svd")(d(a), m, n, d(u), d(s), d(v)))
        return u, s, v

    def sym_eig(self, t):
        t = F(t)
        n = t.shape[0]
        vals = np.zeros(n)
        vecs = np.zeros((n, n), order="F")
        self._chk(self.f("sym_eig")(d(t), n, d(vals), d(vecs)))
        return vals, vecs

    def sample(self, a, l, q, s, r, left=False):
        a = F(a)
        m, n = a.shape
        y = np.zeros((l, n) if left else (m, l), order="F")
        if self.p == "orc_":
            fn = self.f("sample_left" if left else "sample_right")
            st = fn(d(a), m, n, l, q, s, C.byref(r), d(y))
        else:
            st = self.f("sample")(int(left), d(a), m, n, l, q, s, C.byref(r), d(y))
        self._chk(st)
        return y

    def rsvd(self, a, k, p, q, s, r, variant=0):
        a = F(a)
        m, n = a.shape
        u = np.zeros((m, k), order="F")
        sg = np.zeros(k)
        v = np.zeros((n, k), order="F")
        self._chk(self.f("rsvd")(variant, d(a), m, n, k, p, q, s, C.byref(r), d(u), d(sg), d(v)))
        return u, sg, v

    def qb_blocked(self, a, b, M, tol, q, reorth, r, want_w=False):
        a = F(a)
        m, n = a.shape
        cap = max(1, min(b * M, min(m, n)))
        Q = np.zeros((m, cap), order="F")
        B = np.zeros((cap, n), order="F")
        hist = np.zeros(M)
        ell, nh, reached = C.c_int(0), C.c_int(0), C.c_int(0)
        fin = C.c_double(0)
        w = np.zeros((m, n), order="F") if want_w else None
        self._chk(self.f("qb_blocked")(d(a), m, n, b, M, C.c_double(tol), q, reorth, C.byref(r),
                                       d(Q), d(B), cap, C.byref(ell), d(hist), C.byref(nh),
                                       C.byref(fin), C.byref(reached),
                                       d(w) if want_w else None))
        e = ell.value
        return dict(q=Q[:, :e].copy(order="F"), b=B[:e].copy(order="F"), ell=e,
                    history=hist[:nh.value].copy(), final=fin.value, reached=bool(reached.value),
                    w=w)

    def svd_from_qb(self, q, b, k=0, vnum=0):
        q, b = F(q), F(b)
        m, ell = q.shape
        n = b.shape[1]
        kk = ell if k == 0 else k
        u = np.zeros((m, max(kk, 1)), order="F")
        s = np.zeros(max(kk, 1))
        v = np.zeros((n, max(kk, 1)), order="F")
        ko = C.c_int(0)
        self._chk(self.f("svd_from_qb")(d(q), d(b), max(ell, 1), m, n, ell, k, vnum, d(u), d(s),
                                        d(v), C.byref(ko)))
        kk = ko.value
        return u[:, :kk], s[:kk], v[:, :kk]

    def id_column(self, a, k, tol=0.0):
        a = F(a)
        m, n = a.shape
        kcap = min(m, n) if k == 0 else k
        jc = np.zeros(n, dtype=np.int32)
        v = np.zeros((n, max(kcap, 1)), order="F")
        ko, reached, cl = C.c_int(0), C.c_int(0), C.c_int(0)
        res = C.c_double(0)
        self._chk(self.f("id_column")(d(a), m, n, k, C.c_double(tol), i(jc), d(v), C.byref(ko),
                                      C.byref(res), C.byref(reached), C.byref(cl)))
        kk = ko.value
        return dict(jc=jc, v=v[:, :kk], k=kk, qr_residual=res.value, reached=bool(reached.value),
                    clamped=bool(cl.value))

    def id_rand(self, a, k, p, q, s, r):
        a = F(a)
        m, n = a.shape
        jc = np.zeros(n, dtype=np.int32)
        v = np.zeros((n, k), order="F")
        res = C.c_double(0)
        cl = C.c_int(0)
        self._chk(self.f("id_rand")(d(a), m, n, k, p, q, s, C.byref(r), i(jc), d(v), C.byref(res),
                                    C.byref(cl)))
        return dict(jc=jc, v=v, qr_residual=res.value, clamped=bool(cl.value))

    def cur_rand(self, a, k, p, q, s, r):
        a = F(a)
        m, n = a.shape
        jc = np.zeros(n, dtype=np.int32)
        jr = np.zeros(m, dtype=np.int32)
        c = np.zeros((m, k), order="F")
        u = np.zeros((k, k), order="F")
        rr = np.zeros((k, n), order="F")
        res, qres = C.c_double(0), C.c_double(0)
        if self.p == "orc_":
            v = np.zeros((n, k), order="F")
            w = np.zeros((m, k), order="F")
            st = self.f("cur_rand")(d(a), m, n, k, p, q, s, C.byref(r), i(jc), i(jr), d(v), d(w),
                                    d(c), d(u), d(rr), C.byref(res), C.byref(qres))
        else:
            st = self.f("cur_rand")(d(a), m, n, k, p, q, s, C.byref(r), i(jc), i(jr), d(c), d(u),
                                    d(rr), C.byref(res), C.byref(qres))
        self._chk(st)
        return dict(jc=jc, jr=jr, c=c, u=u, r=rr, residual=res.value, qr_residual=qres.value)

    def two_sided_from_column(self, a, jc, v, k):
        a = F(a)
        m, n = a.shape
        jc = np.ascontiguousarray(jc, dtype=np.int32)
        jr = np.zeros(m, dtype=np.int32)
        w = np.zeros((m, k), order="F")
        if self.p == "orc_":
            st = self.f("two_sided_from_column")(d(a), m, n, i(jc), k, i(jr), d(w))
        else:
            v = F(v)
            st = self.f("two_sided_from_column")(d(a), m, n, i(jc), d(v), k, i(jr), d(w))
        self._chk(st)
        return jr, w


_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        _ensure_built()
        _orc = _Lib(ORC_PATH, "orc_")
        _orc.lib.orc_last_error.restype = C.c_char_p
    return _orc


def have_ref():
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        _ref = _Lib(REF_PATH, "ref_")
        _ref.lib.ref_last_error.restype = C.c_char_p
    return _ref
