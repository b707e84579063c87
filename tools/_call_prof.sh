set -x
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_algorithms.py -q -x -p no:cacheprovider > gpurun_out/p6_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/p6_tests.log
python - <<'PY'
import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_1502_05366_b200 as R
eng = R.Engine(0)
for (m, n) in [(610, 10000), (600, 20000)]:
    a = np.random.default_rng(0).standard_normal((m, n))
    eng.pivoted_qr_partial(a, 600)
    eng.profile(True)
    t0 = time.perf_counter(); eng.pivoted_qr_partial(a, 600); t1 = time.perf_counter()
    rec = [r for r in eng.profile_records() if r["name"] == "cpqr"]
    eng.profile(False)
    print(m, n, "pivoted_qr_partial (with Q1) ms", rec[-1]["ms"], "wall", 1e3 * (t1 - t0))
for (m, n, r) in [(610, 600, 300), (2000, 210, 100), (20000, 500, 200)]:
    rs = np.random.default_rng(1)
    a = rs.standard_normal((m, r)) @ rs.standard_normal((r, n))
    eng.orth(a)
    t0 = time.perf_counter(); q = eng.orth(a); t1 = time.perf_counter()
    print(m, n, "rank", r, "orth (Householder fallback) wall ms", 1e3 * (t1 - t0), "defect", np.linalg.norm(q.T @ q - np.eye(n)))
PY
