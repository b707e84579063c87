"""C1 latency anatomy: the small SVD of a C1-shaped R-hat (l = 210, spectrum
exp(-j/20)) and the l x l Cholesky, with the kernels' phase clocks
(RLRA_JACOBI_PHASES / RLRA_CHOL_PROBE set by the caller).  Prints one line
per measurement."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1502_05366_b200 as R

l = int(os.environ.get("L", 210))
dec = float(os.environ.get("DECAY", 20.0))
rs = np.random.default_rng(0)
Q, _ = np.linalg.qr(rs.standard_normal((l, l)))
sig = np.exp(-np.arange(l) / dec)
a = np.triu(np.linalg.qr((Q * sig) @ np.linalg.qr(rs.standard_normal((l, l)))[0].T)[1])
eng = R.Engine(0)
for it in range(3):
    eng.profile(True)
    t0 = time.perf_counter()
    u, s, v = eng.small_svd(a)
    t1 = time.perf_counter()
    recs = eng.profile_records()
    eng.profile(False)
    err = np.max(np.abs(s - sig) / sig)
    print(f"small_svd l={l} wall {1e3*(t1-t0):.3f} ms rel_err {err:.2e}",
          [(r['name'], round(r['ms'], 3), r['K']) for r in recs], flush=True)
g = a.T @ a
for it in range(3):
    eng.profile(True)
    t0 = time.perf_counter()
    eng.orth(np.asfortranarray(rs.standard_normal((2000, l))))
    t1 = time.perf_counter()
    recs = eng.profile_records()
    eng.profile(False)
    print(f"orth 2000x{l} wall {1e3*(t1-t0):.3f} ms", [(r['name'], round(r['ms'], 3)) for r in recs], flush=True)
