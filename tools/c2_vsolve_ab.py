"""C2's svd_from_qb with the R-hat Jacobi's V accumulated (RLRA_SVD_VSOLVE=0,
the reference's arithmetic) or recovered as R^{-1} W (default): device time,
sigma, orthonormality of U and V, and ||A - U S V^T||_F / ||A||_F.  Run once
per mode (the mode is read once per process); argv[1] = output .npz for the
sigma cross-check."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1502_05366_b200 as R
from paper_1502_05366_b200.testmat import gen_test_matrix_device

m = n = int(os.environ.get("N", 8000))
b = 100
M = -(-m // b)
eng = R.Engine(0)
A, s = gen_test_matrix_device(eng, m, n, (np.arange(min(m, n)) + 1.0) ** -2, seed=2)
cap = min(b * M, m)
Q = torch.empty(m * cap, dtype=torch.float64, device="cuda")
B = torch.empty(cap * n, dtype=torch.float64, device="cuda")
f = eng.device_qb_blocked(A.data_ptr(), m, n, m, False, b, M, 1e-6, 1, 1, R.Omega.philox(12345), Q.data_ptr(), m,
                          B.data_ptr(), cap, cap)
ell = f["ell"]
U = torch.empty(m * ell, dtype=torch.float64, device="cuda")
V = torch.empty(n * ell, dtype=torch.float64, device="cuda")
S = torch.empty(ell, dtype=torch.float64, device="cuda")
times = []
for rep in range(2):
    eng.synchronize()
    t0 = time.perf_counter()
    eng.device_svd_from_qb(Q.data_ptr(), m, m, B.data_ptr(), n, cap, ell, 0, 0, U.data_ptr(), m, S.data_ptr(),
                           V.data_ptr(), n)
    eng.synchronize()
    times.append(time.perf_counter() - t0)
Um = U.view(ell, m).T
Vm = V.view(ell, n).T
Am = A.view(n, m).T
I = torch.eye(ell, dtype=torch.float64, device="cuda")
orth_u = (Um.T @ Um - I).abs().max().item()
orth_v = (Vm.T @ Vm - I).abs().max().item()
res = torch.linalg.norm(Am - (Um * S) @ Vm.T).item() / torch.linalg.norm(Am).item()
sv = S.cpu().numpy()
st = s.cpu().numpy()[:ell]
if len(sys.argv) > 1:
    np.savez(sys.argv[1], s=sv)
print(json.dumps(dict(mode=os.environ.get("RLRA_SVD_VSOLVE", "1"), ell=ell, svd_s=times, orth_u=orth_u,
                      orth_v=orth_v, rel_resid=res, qb_final=f["final_residual"],
                      top100_rel_vs_true=float(np.max(np.abs(sv[:100] - st[:100]) / st[:100])))), flush=True)
