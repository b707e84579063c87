"""small_svd of an l x l graded upper-triangular matrix (the R-hat of
rsvd_v2): SPEC=exp (C5: exp(-j/100)) or SPEC=sqrt (C4: 1/sqrt(j+1) plus a
0.45-level noise floor).  Prints wall/device ms and the sweeps used."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1502_05366_b200 as R
l = int(os.environ.get("L", 510))
spec = os.environ.get("SPEC", "exp")
rs = np.random.default_rng(0)
Q, _ = np.linalg.qr(rs.standard_normal((l, l)))
sig = np.exp(-np.arange(l) / 100.0) if spec == "exp" else np.sqrt(1.0 / (np.arange(l) + 1.0) + 0.2)
a = np.triu(np.linalg.qr((Q * sig) @ np.linalg.qr(rs.standard_normal((l, l)))[0].T)[1])
eng = R.Engine(0)
eng.small_svd(a)
eng.profile(True)
t0 = time.perf_counter()
u, s, v = eng.small_svd(a)
t1 = time.perf_counter()
recs = eng.profile_records()
err = np.max(np.abs(s - np.sort(sig)[::-1]) / np.sort(sig)[::-1])
print(f"l={l} spec={spec} wall {1e3*(t1-t0):.2f} ms sigma_rel_err {err:.2e}",
      [(r['name'], round(r['ms'], 3), r['K']) for r in recs], flush=True)
