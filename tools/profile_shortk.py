"""The short-K NN product of CholQR / the lift at C5 shapes: Y (200000 x 510)
times a 510 x 510 matrix, for ncu (-k regex:dgemm_tma --launch-skip 1 -c 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1502_05366_b200 as R

m, l = 200000, 510
eng = R.Engine(0)
Y = torch.empty(m * l, dtype=torch.float64, device="cuda")
B = torch.empty(l * l, dtype=torch.float64, device="cuda")
Q = torch.empty(m * l, dtype=torch.float64, device="cuda")
eng.device_gaussian_philox(m, l, 1, 0, 0, Y.data_ptr(), m)
eng.device_gaussian_philox(l, l, 2, 0, 0, B.data_ptr(), l)
for _ in range(2):
    eng.device_matmul(False, False, Y.data_ptr(), m, l, m, B.data_ptr(), l, l, l, Q.data_ptr(), m)
eng.synchronize()
print("ok")
