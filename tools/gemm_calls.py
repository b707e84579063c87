"""Every profiled call of one rsvd_v2 at C1 (2000 x 4000, k = 200, p = 10,
q = 2; default) or C5 (argument "C5": 200000 x 20000, k = 500, p = 10,
q = 2), or of one id_rand at C3 (argument "C3": 20000 x 10000, k = 600),
with its shape and device ms: where the time goes, GEMM by GEMM."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1502_05366_b200 as R
from paper_1502_05366_b200.testmat import gen_test_matrix_device

eng = R.Engine(0)
cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
if cfg == "C3":
    m, n, k, p, q = 20000, 10000, 600, 10, 2
    A, _ = gen_test_matrix_device(eng, m, n, 10.0 ** (-8.0 * np.arange(1500) / 1500), seed=3, noise=1e-10)
    jc = torch.empty(n, dtype=torch.int32, device="cuda")
    V = torch.empty(n * k, dtype=torch.float64, device="cuda")
    run = lambda: eng.device_id_rand(A.data_ptr(), m, n, m, k, p, q, 1, R.Omega.philox(12345), jc.data_ptr(),
                                     V.data_ptr(), n)
else:
    m, n, k, p, q, dec = (200000, 20000, 500, 10, 2, 100.0) if cfg == "C5" else (2000, 4000, 200, 10, 2, 20.0)
    A, _ = gen_test_matrix_device(eng, m, n, np.exp(-np.arange(min(m, n)) / dec), seed=1)
    U = torch.empty(m * k, dtype=torch.float64, device="cuda")
    V = torch.empty(n * k, dtype=torch.float64, device="cuda")
    S = torch.empty(k, dtype=torch.float64, device="cuda")
    run = lambda: eng.device_rsvd(R.RSVD_V2, A.data_ptr(), m, n, m, k, p, q, 1, R.Omega.philox(12345),
                                  U.data_ptr(), S.data_ptr(), V.data_ptr())
run()
eng.synchronize()
eng.profile(True)
run()
eng.synchronize()
recs = eng.profile_records()
eng.profile(False)
for r in recs:
    print(f"{r['name']:12s} M={r['M']:6d} N={r['N']:6d} K={r['K']:6d} {r['ms']*1e3:8.1f} us"
          + (f" {r['flops'] / r['ms'] / 1e9:6.2f} TF/s" if r['flops'] > 0 else ""))
