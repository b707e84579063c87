"""A/B of small_svd on one fixed C2-like R-hat (6100 x 6100) between the
current library and an alternative build (argv[1]: path of the .so), same
input bits: prints device ms and sweeps for each."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1502_05366_b200 as R

alt = sys.argv[1] if len(sys.argv) > 1 else None
if alt:
    R.LIB_PATH = alt
n = 6100
rs = np.random.default_rng(0)
# a graded upper-triangular matrix with the C2 spectrum (j+1)^-2
q, _ = np.linalg.qr(rs.standard_normal((n, n)))
r = np.triu(np.linalg.qr((q * ((np.arange(n) + 1.0) ** -2)) @ np.linalg.qr(rs.standard_normal((n, n)))[0].T)[1])
eng = R.Engine(0)
eng.profile(True)
u, s, v = eng.small_svd(r)
rec = [x for x in eng.profile_records() if x["name"] == "small_svd"][-1]
print(json.dumps({"lib": alt or "current", "svd_ms": round(rec["ms"], 1), "sweeps": rec["K"]}), flush=True)
