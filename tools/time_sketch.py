import os, sys, json
sys.path.insert(0, "/root/repo")
import torch
import paper_1502_05366_b200 as R
m, n, l = 200000, 20000, 510
eng = R.Engine(0)
A = torch.empty(m * n, dtype=torch.float64, device="cuda")
Y = torch.empty(m * l, dtype=torch.float64, device="cuda")
eng.device_gaussian_philox(m, n, 1, 0, 0, A.data_ptr(), m)
st = torch.cuda.ExternalStream(eng.stream)
fn = lambda: eng.device_sketch(False, A.data_ptr(), m, n, m, l, R.Omega.philox(3), 0, 0, Y.data_ptr(), m)
fn(); eng.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(3): fn()
e1.record(st); e1.synchronize()
ms = e0.elapsed_time(e1) / 3
print(json.dumps({"sketch_ms": round(ms, 2), "tflops": round(2.0 * m * n * l / ms / 1e9, 2)}))
