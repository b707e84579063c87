"""Every profiled call of one C2 qb_blocked (8000 x 8000, b = 100, tol 1e-6,
q = 1), summed by (name, shape): where the QB time goes."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1502_05366_b200 as R
from paper_1502_05366_b200.testmat import gen_test_matrix_device

eng = R.Engine(0)
m = n = 8000
b, M = 100, 80
A, _ = gen_test_matrix_device(eng, m, n, (np.arange(m) + 1.0) ** -2, seed=2)
cap = b * M
Q = torch.empty(m * cap, dtype=torch.float64, device="cuda")
B = torch.empty(cap * n, dtype=torch.float64, device="cuda")
W = torch.empty_like(A)


def run():
    W.copy_(A)
    return eng.device_qb_blocked(W.data_ptr(), m, n, m, True, b, M, 1e-6, 1, 1, R.Omega.philox(12345), Q.data_ptr(),
                                 m, B.data_ptr(), cap, cap)


run()
eng.synchronize()
eng.profile(True)
f = run()
eng.synchronize()
recs = eng.profile_records()
eng.profile(False)
agg = defaultdict(lambda: [0, 0.0, 0.0])
for r in recs:
    key = (r["name"], r["M"], r["N"], r["K"])
    agg[key][0] += 1
    agg[key][1] += r["ms"]
    agg[key][2] += r["flops"]
print("ell", f["ell"])
for key, (cnt, ms, fl) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{key[0]:12s} M={key[1]:5d} N={key[2]:5d} K={key[3]:5d} x{cnt:3d} {ms:8.2f} ms" +
          (f" {fl / ms / 1e9:6.2f} TF/s" if fl > 0 else ""))
