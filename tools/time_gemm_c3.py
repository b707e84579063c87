"""CUDA-event times of C3's A-streaming products (TN: 10000 x 610, k = 20000;
NN: 20000 x 610, k = 10000) on the engine stream — or C1's (2000 x 4000,
l = 210) with SHAPE=C1; RLRA_GEMM_SPLITS forces a split-K count for A/B
runs.  Prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1502_05366_b200 as R

m, n, l = (2000, 4000, 210) if os.environ.get("SHAPE") == "C1" else (20000, 10000, 610)
eng = R.Engine(0)
st = torch.cuda.ExternalStream(eng.stream)
A = torch.empty(m * n, dtype=torch.float64, device="cuda")
Y = torch.empty(m * l, dtype=torch.float64, device="cuda")
Z = torch.empty(n * l, dtype=torch.float64, device="cuda")
eng.device_gaussian_philox(m, n, 1, 0, 0, A.data_ptr(), m)
eng.device_gaussian_philox(m, l, 2, 0, 0, Y.data_ptr(), m)
eng.device_gaussian_philox(n, l, 3, 0, 0, Z.data_ptr(), n)
out = {"splits": os.environ.get("RLRA_GEMM_SPLITS", "auto")}
for name, fn in (("TN", lambda: eng.device_matmul(True, False, A.data_ptr(), m, n, m, Y.data_ptr(), m, l, m,
                                                  Z.data_ptr(), n)),
                 ("NN", lambda: eng.device_matmul(False, False, A.data_ptr(), m, n, m, Z.data_ptr(), n, l, n,
                                                  Y.data_ptr(), m))):
    fn()
    eng.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(20):
        fn()
    e1.record(st)
    e1.synchronize()
    out[name + "_ms"] = round(e0.elapsed_time(e1) / 20, 3)
print(json.dumps(out), flush=True)
