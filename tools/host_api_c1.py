"""C1 (2000 x 4000, k = 200, p = 10, q = 2) through the public host API the
way a reference user calls it: A in a pageable numpy array, Philox Omega,
wall time per call (upload, compute, U/sigma/V download) after a warm-up,
against the device-resident call."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1502_05366_b200 as R

eng = R.Engine(0)
m, n, k, p, q = 2000, 4000, 200, 10, 2
rs = np.random.default_rng(1)
u, _ = np.linalg.qr(rs.standard_normal((m, m)))
v, _ = np.linalg.qr(rs.standard_normal((n, m)))
a = np.asfortranarray((u * np.exp(-np.arange(m) / 20.0)) @ v.T)
om = R.Omega.philox(12345)
for _ in range(3):
    eng.rsvd_v2(a, k, p, q, 1, omega=om)
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    U, S, V = eng.rsvd_v2(a, k, p, q, 1, omega=om)
    ts.append(time.perf_counter() - t0)
print(json.dumps({"config": "C1 host API (pageable numpy A)", "median_ms": 1e3 * float(np.median(ts)),
                  "min_ms": 1e3 * min(ts), "sigma0": float(S[0])}))
eng.profile(True)
t0 = time.perf_counter()
eng.rsvd_v2(a, k, p, q, 1, omega=om)
t1 = time.perf_counter()
recs = eng.profile_records()
eng.profile(False)
print("wall ms", round(1e3 * (t1 - t0), 3), "device phases:",
      [(r["name"], r["M"], r["N"], r["K"], round(r["ms"], 3)) for r in recs if r["name"] not in ("gemm_orth", "chol")])
# the C call alone with pre-touched outputs (no fresh-page faults in the download)
import ctypes as C
from paper_1502_05366_b200 import lib, HOST, RSVD_V2, _d, _i64, _check
u = np.ones((m, k), order="F"); sg = np.ones(k); vv = np.ones((n, k), order="F")
ts = []
for _ in range(10):
    st = om.struct()
    t0 = time.perf_counter()
    _check(lib().rlra_rsvd(eng._ctx, HOST, RSVD_V2, _d(a), m, n, _i64(m), k, p, q, 1, C.byref(st), _d(u), _i64(m),
                           _d(sg), _d(vv), _i64(n)))
    ts.append(time.perf_counter() - t0)
t0 = time.perf_counter()
for _ in range(10):
    x = np.zeros((m, k), order="F"); y = np.zeros((n, k), order="F"); x[:] = 1.0; y[:] = 1.0
t1 = time.perf_counter()
print(json.dumps({"C call, pre-touched outputs, median ms": 1e3 * float(np.median(ts)),
                  "fresh output alloc+touch ms": 1e3 * (t1 - t0) / 10}))
