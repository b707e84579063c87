"""small_svd of an l x l graded upper-triangular matrix (the R-hat of rsvd_v2 at C5)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1502_05366_b200 as R
l = int(os.environ.get("L", 510))
rs = np.random.default_rng(0)
Q, _ = np.linalg.qr(rs.standard_normal((l, l)))
a = np.triu(np.linalg.qr((Q * np.exp(-np.arange(l) / 100.0)) @ np.linalg.qr(rs.standard_normal((l, l)))[0].T)[1])
eng = R.Engine(0)
eng.small_svd(a)
eng.profile(True)
t0 = time.perf_counter()
u, s, v = eng.small_svd(a)
t1 = time.perf_counter()
recs = eng.profile_records()
print(f"l={l} wall {1e3*(t1-t0):.2f} ms", [(r['name'], round(r['ms'], 3), r['K']) for r in recs])
