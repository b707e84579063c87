"""Time the dominant C5 GEMM shapes with CUDA events (engine stream).
Usage: RLRA_GEMM_CFG=w8|w16 python tools/gemm_tune.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1502_05366_b200 as R

m, n, l = int(os.environ.get("M", 200000)), int(os.environ.get("N", 20000)), int(os.environ.get("L", 510))
eng = R.Engine(0)
A = torch.empty(m * n, dtype=torch.float64, device="cuda")
Z = torch.empty(n * l, dtype=torch.float64, device="cuda")
Y = torch.empty(m * l, dtype=torch.float64, device="cuda")
eng.device_gaussian_philox(m, n, 1, 0, 0, A.data_ptr(), m)
eng.device_gaussian_philox(n, l, 2, 0, 0, Z.data_ptr(), n)
st = torch.cuda.ExternalStream(eng.stream)
res = {"cfg": os.environ.get("RLRA_GEMM_CFG", "default")}
for name, fn in [("NN", lambda: eng.device_matmul(False, False, A.data_ptr(), m, n, m, Z.data_ptr(), n, l, n, Y.data_ptr(), m)),
                 ("TN", lambda: eng.device_matmul(True, False, A.data_ptr(), m, n, m, Y.data_ptr(), m, l, m, Z.data_ptr(), n))]:
    fn(); eng.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record(st)
    for _ in range(reps): fn()
    e1.record(st); e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[name] = dict(ms=round(ms, 2), tflops=round(2.0 * m * n * l / ms / 1e9, 2))
print(json.dumps(res))
