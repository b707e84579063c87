"""Every profiled call of one C3 cur_rand (20000 x 10000, k = 600, p = 10,
q = 2, device buffers) with its shape and device ms."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1502_05366_b200 as R
from paper_1502_05366_b200.testmat import gen_test_matrix_device

eng = R.Engine(0)
m, n, k, p, q = 20000, 10000, 600, 10, 2
A, _ = gen_test_matrix_device(eng, m, n, 10.0 ** (-8.0 * np.arange(1500) / 1500), seed=3, noise=1e-10)
dev = {"jc": torch.empty(n, dtype=torch.int32, device="cuda"), "jr": torch.empty(m, dtype=torch.int32, device="cuda"),
       "v": torch.empty(n * k, dtype=torch.float64, device="cuda"), "w": torch.empty(m * k, dtype=torch.float64, device="cuda"),
       "c": torch.empty(m * k, dtype=torch.float64, device="cuda"), "u": torch.empty(k * k, dtype=torch.float64, device="cuda"),
       "r": torch.empty(k * n, dtype=torch.float64, device="cuda")}
ptrs = {key: t.data_ptr() for key, t in dev.items()}
run = lambda: eng.device_cur_rand(A.data_ptr(), m, n, m, k, p, q, 1, R.Omega.philox(12345), ptrs)
run()
eng.synchronize()
eng.profile(True)
run()
eng.synchronize()
recs = eng.profile_records()
eng.profile(False)
tot = {}
for r in recs:
    print(f"{r['name']:12s} M={r['M']:6d} N={r['N']:6d} K={r['K']:6d} {r['ms']*1e3:9.1f} us")
