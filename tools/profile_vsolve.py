"""Where svd_vsolve's time goes at C2 (the R-hat V recovery): the profiled
calls recorded after the svd_vsolve scope opens, in order, summed by name
and K (the blocked solve's GEMMs have K = 64)."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1502_05366_b200 as R
from paper_1502_05366_b200.testmat import gen_test_matrix_device

m = n = 8000
b, M = 100, 80
eng = R.Engine(0)
A, s = gen_test_matrix_device(eng, m, n, (np.arange(n) + 1.0) ** -2, seed=2)
Q = torch.empty(m * m, dtype=torch.float64, device="cuda")
B = torch.empty(m * n, dtype=torch.float64, device="cuda")
f = eng.device_qb_blocked(A.data_ptr(), m, n, m, False, b, M, 1e-6, 1, 1, R.Omega.philox(12345), Q.data_ptr(), m,
                          B.data_ptr(), m, m)
ell = f["ell"]
U = torch.empty(m * ell, dtype=torch.float64, device="cuda")
V = torch.empty(n * ell, dtype=torch.float64, device="cuda")
S = torch.empty(ell, dtype=torch.float64, device="cuda")
eng.profile(True)
eng.device_svd_from_qb(Q.data_ptr(), m, m, B.data_ptr(), n, m, ell, 0, 0, U.data_ptr(), m, S.data_ptr(),
                       V.data_ptr(), n)
eng.synchronize()
recs = eng.profile_records()
i0 = next(i for i, r in enumerate(recs) if r["name"] == "svd_vsolve")
print(f"svd_vsolve {recs[i0]['ms']:.2f} ms")
agg = collections.OrderedDict()
for r in recs[i0 + 1:]:
    if r["name"] == "gemm_lift":
        break
    key = (r["name"], r["K"] if r["K"] == 64 else (r["M"], r["N"], r["K"]))
    c, t = agg.get(key, (0, 0.0))
    agg[key] = (c + 1, t + r["ms"])
for k, (c, t) in agg.items():
    print(f"{k}: {c} calls, {t:.2f} ms")
