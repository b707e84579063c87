"""Run the dominant C5 GEMMs once each (for ncu --set full):
   Y = A Omega  (NN, Philox Omega in-register; 200000 x 510, K = 20000) — sketch
   Y = A Z      (NN, 200000 x 510, K = 20000)                           — power products
   Z = A^T Y    (TN, 20000 x 510, K = 200000)                           — power / projection
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1502_05366_b200 as R

m, n, l = int(os.environ.get("M", 200000)), int(os.environ.get("N", 20000)), 510
eng = R.Engine(0)
A = torch.empty(m * n, dtype=torch.float64, device="cuda")
Z = torch.empty(n * l, dtype=torch.float64, device="cuda")
Y = torch.empty(m * l, dtype=torch.float64, device="cuda")
eng.device_gaussian_philox(m, n, 1, 0, 0, A.data_ptr(), m)
eng.device_gaussian_philox(n, l, 2, 0, 0, Z.data_ptr(), n)
eng.device_sketch(False, A.data_ptr(), m, n, m, l, R.Omega.philox(3), 0, 0, Y.data_ptr(), m)
eng.device_matmul(False, False, A.data_ptr(), m, n, m, Z.data_ptr(), n, l, n, Y.data_ptr(), m)
eng.device_matmul(True, False, A.data_ptr(), m, n, m, Y.data_ptr(), m, l, m, Z.data_ptr(), n)
eng.synchronize()
print("ok")
