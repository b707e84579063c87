"""C1 through the host API from a pageable numpy A and from a pinned (torch
pin_memory) view of the same matrix, plus torch's own 64 MB copies for scale;
RLRA_HOSTIO_TIMES=1 prints the host-path marks and the staged pieces."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1502_05366_b200 as R
eng = R.Engine(0)
m, n, k, p, q = 2000, 4000, 200, 10, 2
a = np.asfortranarray(np.random.default_rng(1).standard_normal((m, n)))
tp = torch.empty(n * m, dtype=torch.float64).pin_memory()
ap = tp.numpy().reshape(n, m).T  # Fortran view, pinned
ap[:] = a
om = R.Omega.philox(12345)
for arr, name in ((a, "pageable"), (ap, "pinned")):
    for _ in range(3): eng.rsvd_v2(arr, k, p, q, 1, omega=om)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); eng.rsvd_v2(arr, k, p, q, 1, omega=om); ts.append(time.perf_counter() - t0)
    print(name, "median ms", 1e3 * float(np.median(ts)), flush=True)
x = torch.from_numpy(a.ravel(order="F").copy())
for src, name in ((x, "torch pageable"), (tp, "torch pinned")):
    for _ in range(3): y = src.cuda(); torch.cuda.synchronize()
    t = time.perf_counter(); y = src.cuda(non_blocking=True); torch.cuda.synchronize(); print(name, "64MB h2d ms", 1e3 * (time.perf_counter() - t))
