"""Time the one-launch cooperative Cholesky + inverse (chol_inv_coop_kernel)
at the rsvd Gram sizes for the grid size in RLRA_CHOL_GRID (device buffers,
CUDA events on the engine stream).  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1502_05366_b200 as R

eng = R.Engine(0)
st = torch.cuda.ExternalStream(eng.stream)
out = {"grid": os.environ.get("RLRA_CHOL_GRID", "default")}
for n in (100, 210, 510, 1020):
    rs = np.random.default_rng(n)
    y = rs.standard_normal((4 * n, n)) * np.exp(-np.arange(n) / (n / 4))
    g = y.T @ y
    eng.chol_inv(g)  # warm
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import time
    t0 = time.perf_counter()
    for _ in range(20):
        eng.chol_inv(g)
    out[f"n{n}_ms_host_api"] = round((time.perf_counter() - t0) / 20 * 1e3, 4)
eng.profile(True)
for n in (100, 210, 510, 1020):
    rs = np.random.default_rng(n)
    y = rs.standard_normal((4 * n, n)) * np.exp(-np.arange(n) / (n / 4))
    g = y.T @ y
    for _ in range(5):
        eng.chol_inv(g)
recs = [r for r in eng.profile_records() if r["name"] == "chol"]
by = {}
for r in recs:
    by.setdefault(r["M"], []).append(r["ms"])
out.update({f"n{k}_ms": round(float(np.median(v)), 4) for k, v in by.items()})
print(json.dumps(out), flush=True)
