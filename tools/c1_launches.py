"""One C1 rsvd_v2 (device-resident, Philox) after a warm-up, bracketed by
markers, for an ncu launch list: the kernels' summed time against the call's
CUDA-event time shows how much of C1 is launch/sync gaps."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1502_05366_b200 as R
from paper_1502_05366_b200.testmat import gen_test_matrix_device

eng = R.Engine(0)
m, n, k, p, q = 2000, 4000, 200, 10, 2
A, _ = gen_test_matrix_device(eng, m, n, np.exp(-np.arange(m) / 20.0), seed=1)
U = torch.empty(m * k, dtype=torch.float64, device="cuda")
V = torch.empty(n * k, dtype=torch.float64, device="cuda")
S = torch.empty(k, dtype=torch.float64, device="cuda")
run = lambda: eng.device_rsvd(R.RSVD_V2, A.data_ptr(), m, n, m, k, p, q, 1, R.Omega.philox(12345), U.data_ptr(),
                              S.data_ptr(), V.data_ptr())
run()
eng.synchronize()
l0 = eng.launches
st = torch.cuda.ExternalStream(eng.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
run()
e1.record(st)
e1.synchronize()
print(json.dumps({"launches_last_call": eng.launches - l0, "call_ms": e0.elapsed_time(e1)}))
