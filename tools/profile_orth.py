"""Time the CholQR pieces at C5 shapes: orth of Y (200000 x 510) and of
Z (20000 x 510), and chol_inv of a 510 x 510 Gram, with the engine's
per-phase CUDA-event records.  Usage: python tools/profile_orth.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1502_05366_b200 as R

m, n, l = int(os.environ.get("M", 200000)), int(os.environ.get("N", 20000)), int(os.environ.get("L", 510))
eng = R.Engine(0)
Y = torch.empty(m * l, dtype=torch.float64, device="cuda")
Z = torch.empty(n * l, dtype=torch.float64, device="cuda")
G = torch.empty(l * l, dtype=torch.float64, device="cuda")
Rm = torch.empty(l * l, dtype=torch.float64, device="cuda")
Ri = torch.empty(l * l, dtype=torch.float64, device="cuda")
st = torch.cuda.ExternalStream(eng.stream)
out = {}
for rep in range(3):
    eng.device_gaussian_philox(m, l, 1, rep, 0, Y.data_ptr(), m)
    eng.device_gaussian_philox(n, l, 2, rep, 0, Z.data_ptr(), n)
    eng.device_gram(Y.data_ptr(), m, l, m, G.data_ptr(), l)
    eng.synchronize()
    eng.profile(True)
    e0, e1, e2, e3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
    e0.record(st)
    eng.device_chol_inv(G.data_ptr(), l, l, 1e-12, Rm.data_ptr(), l, Ri.data_ptr(), l)
    e1.record(st)
    eng.device_orth(Y.data_ptr(), m, l)
    e2.record(st)
    eng.device_orth(Z.data_ptr(), n, l)
    e3.record(st)
    e3.synchronize()
    recs = eng.profile_records()
    eng.profile(False)
    ph = {}
    for r in recs:
        ph[r["name"]] = round(ph.get(r["name"], 0.0) + r["ms"], 3)
    out[rep] = {"chol_inv_ms": round(e0.elapsed_time(e1), 3), "orth_Y_ms": round(e1.elapsed_time(e2), 3),
                "orth_Z_ms": round(e2.elapsed_time(e3), 3), "phases": ph}
print(json.dumps(out[2]))
