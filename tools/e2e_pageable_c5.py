"""C5 rsvd_v2 end to end through the C-ABI from PAGEABLE host memory (what a
reference user's DenseMatrix is) versus pinned memory: wall time per call
(H2D of A, D2H of U/sigma/V inside), Philox Omega.  Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1502_05366_b200 as R
from paper_1502_05366_b200.testmat import gen_test_matrix_device

m, n, k, p, q = 200000, 20000, 500, 10, 2
eng = R.Engine(0)
A, _ = gen_test_matrix_device(eng, m, n, np.exp(-np.arange(3685) / 100.0), seed=5)
out = {}
for kind in ("pinned", "pageable"):
    Ah = torch.empty(m * n, dtype=torch.float64, pin_memory=kind == "pinned")
    Ah.copy_(A)
    Uh = torch.empty(m * k, dtype=torch.float64, pin_memory=kind == "pinned")
    Vh = torch.empty(n * k, dtype=torch.float64, pin_memory=kind == "pinned")
    Sh = torch.empty(k, dtype=torch.float64, pin_memory=kind == "pinned")
    call = lambda s: eng.host_rsvd_ptr(R.RSVD_V2, Ah.data_ptr(), m, n, m, k, p, q, 1, R.Omega.philox(s),
                                       Uh.data_ptr(), Sh.data_ptr(), Vh.data_ptr())
    call(1)
    ts = []
    for s in range(3):
        t0 = time.perf_counter()
        call(10 + s)
        ts.append(time.perf_counter() - t0)
    out[kind + "_ms"] = 1e3 * min(ts)
    del Ah, Uh, Vh, Sh
out["threads"] = int(os.environ.get("RLRA_UPLOAD_THREADS", os.cpu_count() or 1))
print(json.dumps(out), flush=True)
