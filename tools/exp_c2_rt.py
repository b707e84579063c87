"""Experiment: the C2 R-hat (QR of B^T after qb_blocked at C2) — one-sided
Jacobi on R versus on R1^T, R P = Q1 R1 a column-pivoted QR (Drmac-Veselic
preconditioning): sweeps and time.  Prints JSON lines."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1502_05366_b200 as R
from paper_1502_05366_b200.testmat import gen_test_matrix_device

eng = R.Engine(0)
m = n = int(os.environ.get("N", 8000))
A, st = gen_test_matrix_device(eng, m, n, (np.arange(m) + 1.0) ** -2, seed=2)
cap = min(100 * 80, m)
Q = torch.empty(m * cap, dtype=torch.float64, device="cuda")
B = torch.empty(cap * n, dtype=torch.float64, device="cuda")
f = eng.device_qb_blocked(A.data_ptr(), m, n, m, False, 100, 80, 1e-6, 1, 1, R.Omega.philox(12345), Q.data_ptr(), m,
                          B.data_ptr(), cap, cap)
ell = f["ell"]
Bh = B.view(n, cap)[:, :ell].cpu().numpy()  # B^T (n x ell), column-major B is cap x n
t0 = time.perf_counter()
r = np.linalg.qr(Bh, mode="r")
print(json.dumps({"ell": ell, "host_qr_s": time.perf_counter() - t0}), flush=True)
r = np.triu(r)
import scipy.linalg
t0 = time.perf_counter()
_, r1, piv = scipy.linalg.qr(r, pivoting=True, mode="economic")
print(json.dumps({"host_qrcp_s": time.perf_counter() - t0}), flush=True)
r1 = np.triu(r1)
for name, mat in (("R", r), ("R1^T (QRCP-preconditioned)", np.asfortranarray(r1.T))):
    eng.profile(True)
    t0 = time.perf_counter()
    u, s, v = eng.small_svd(mat)
    dt = time.perf_counter() - t0
    rec = [x for x in eng.profile_records() if x["name"] == "small_svd"]
    eng.profile(False)
    print(json.dumps({"input": name, "wall_s": dt, "svd_ms": rec[-1]["ms"], "sweeps": rec[-1]["K"],
                      "sigma_top_rel_vs_true": float(np.max(np.abs(s[:100] - st.cpu().numpy()[:100]) / st.cpu().numpy()[:100]))}),
          flush=True)
