"""CUDA-event times of the C5 A-streaming GEMMs (NN: Y = A Z, TN: Z = A^T Y)
on the engine stream, 3 repetitions each after a warm-up.  Prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1502_05366_b200 as R

m, n, l = 200000, 20000, 510
eng = R.Engine(0)
st = torch.cuda.ExternalStream(eng.stream)
A = torch.empty(m * n, dtype=torch.float64, device="cuda")
Z = torch.empty(n * l, dtype=torch.float64, device="cuda")
Y = torch.empty(m * l, dtype=torch.float64, device="cuda")
eng.device_gaussian_philox(m, n, 1, 0, 0, A.data_ptr(), m)
eng.device_gaussian_philox(n, l, 2, 0, 0, Z.data_ptr(), n)
out = {}
for name, fn in (("NN", lambda: eng.device_matmul(False, False, A.data_ptr(), m, n, m, Z.data_ptr(), n, l, n,
                                                  Y.data_ptr(), m)),
                 ("TN", lambda: eng.device_matmul(True, False, A.data_ptr(), m, n, m, Y.data_ptr(), m, l, m,
                                                  Z.data_ptr(), n))):
    fn()
    eng.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(3):
        fn()
    e1.record(st)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    out[name + "_ms"] = round(ms, 3)
    out[name + "_tflops"] = round(2.0 * m * n * l / ms / 1e9, 2)
print(json.dumps(out), flush=True)
