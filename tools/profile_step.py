"""One C5 rsvd_v2 step for the per-kernel ncu table (profiles/): generates A
on the GPU, runs one warm-up call, then one profiled call.  Prints the number
of engine launches in the last call so the ncu launch list can be cut to it.
Usage: ncu --metrics ... --csv --log-file X python tools/profile_step.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1502_05366_b200 as R
from paper_1502_05366_b200.testmat import gen_test_matrix_device

m, n, k, p, q = int(os.environ.get("M", 200000)), int(os.environ.get("N", 20000)), 500, 10, 2
eng = R.Engine(0)
A, st = gen_test_matrix_device(eng, m, n, np.exp(-np.arange(3685) / 100.0), seed=5)
U = torch.empty(m * k, dtype=torch.float64, device="cuda")
V = torch.empty(n * k, dtype=torch.float64, device="cuda")
S = torch.empty(k, dtype=torch.float64, device="cuda")


def step(seed):
    eng.device_rsvd(R.RSVD_V2, A.data_ptr(), m, n, m, k, p, q, 1, R.Omega.philox(seed), U.data_ptr(),
                    S.data_ptr(), V.data_ptr())


step(1)
eng.synchronize()
l0 = eng.launches
step(2)
eng.synchronize()
print(json.dumps({"launches_last_call": eng.launches - l0}))
