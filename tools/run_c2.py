"""C2 at full size on one GPU: qb_blocked(b=100, M=80, tol=1e-6, q=1, reorth=1)
then svd_from_qb(k=0) on A = U diag((j+1)^-2) V^T, m=n=8000."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1502_05366_b200 as R
from paper_1502_05366_b200.testmat import gen_test_matrix_device
m = n = int(os.environ.get("N", 8000)); b = 100; M = -(-m // b); tol = float(os.environ.get("TOL", 1e-6))
eng = R.Engine(0)
A, s = gen_test_matrix_device(eng, m, n, (np.arange(min(m, n)) + 1.0) ** -2, seed=2)
cap = min(b * M, m)
Q = torch.empty(m * cap, dtype=torch.float64, device="cuda"); B = torch.empty(cap * n, dtype=torch.float64, device="cuda")
eng.profile(True)
t0 = time.perf_counter()
f = eng.device_qb_blocked(A.data_ptr(), m, n, m, False, b, M, tol, 1, 1, R.Omega.philox(12345), Q.data_ptr(), m, B.data_ptr(), cap, cap)
t1 = time.perf_counter()
ell = f["ell"]
U = torch.empty(m * ell, dtype=torch.float64, device="cuda"); V = torch.empty(n * ell, dtype=torch.float64, device="cuda"); S = torch.empty(ell, dtype=torch.float64, device="cuda")
k = eng.device_svd_from_qb(Q.data_ptr(), m, m, B.data_ptr(), n, cap, ell, 0, 0, U.data_ptr(), m, S.data_ptr(), V.data_ptr(), n)
t2 = time.perf_counter()
ph = {}
for r in eng.profile_records():
    ph[r["name"]] = ph.get(r["name"], 0) + r["ms"]
sv = S.cpu().numpy(); st = s.cpu().numpy()
print(json.dumps(dict(ell=ell, blocks=len(f["history"]), final=f["final_residual"], reached=f["tolerance_reached"],
      qb_s=t1 - t0, svd_s=t2 - t1, top100_rel=float(np.max(np.abs(sv[:100] - st[:100]) / st[:100])),
      phases={k_: round(v_, 1) for k_, v_ in ph.items()},
      sweeps=[r["K"] for r in eng.profile_records() if r["name"] == "small_svd"])))
