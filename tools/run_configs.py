"""Time every BASELINE.json config on one B200 (the bench line covers C5;
this is the per-config table of SURVEY.md §8d): device-resident A generated
on the GPU with the configs' spectra (paper_1502_05366_b200.testmat), Philox
Omega, CUDA-event times on the engine stream, and the accuracy against the
known spectrum.  Usage: python tools/run_configs.py [C1 C2 ...]
Prints one JSON line per config."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1502_05366_b200 as R
from paper_1502_05366_b200.testmat import gen_test_matrix_device

eng = R.Engine(0)
stream = torch.cuda.ExternalStream(eng.stream)


def timed(fn, reps=1):
    fn()
    eng.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def phases(fn):
    """Per-phase device ms of one call (engine profile records; nested)."""
    eng.profile(True)
    fn()
    eng.synchronize()
    out = {}
    for r in eng.profile_records():
        out[r["name"]] = round(out.get(r["name"], 0.0) + r["ms"], 3)
    eng.profile(False)
    return out


def rsvd_cfg(name, m, n, k, p, q, sigma, noise=0.0, seed=1, reps=3):
    A, st = gen_test_matrix_device(eng, m, n, sigma, seed=seed, noise=noise)
    U = torch.empty(m * k, dtype=torch.float64, device="cuda")
    V = torch.empty(n * k, dtype=torch.float64, device="cuda")
    S = torch.empty(k, dtype=torch.float64, device="cuda")

    def run():
        eng.device_rsvd(R.RSVD_V2, A.data_ptr(), m, n, m, k, p, q, 1, R.Omega.philox(12345),
                        U.data_ptr(), S.data_ptr(), V.data_ptr())

    t = timed(run, reps)
    ph = phases(run)
    l = k + p
    F = 4.0 * m * n * l * (q + 1)
    rel = eng.device_rel_error(A.data_ptr(), m, n, U.data_ptr(), S.data_ptr(), V.data_ptr(), k)
    s = S.cpu().numpy()
    top = min(20, k)
    stt = st.cpu().numpy()[:top]
    return dict(config=name, entry="rsvd_v2", m=m, n=n, k=k, p=p, q=q, time_s=t, tflops=F / t / 1e12,
                rel_fro_error=rel, sigma_top20_rel_vs_true=float(np.max(np.abs(s[:top] - stt) / stt)), phases_ms=ph)


def c2():
    m = n = 8000
    b, M, tol = 100, 80, 1e-6
    A, st = gen_test_matrix_device(eng, m, n, (np.arange(m) + 1.0) ** -2, seed=2)
    cap = min(b * M, m)
    Q = torch.empty(m * cap, dtype=torch.float64, device="cuda")
    B = torch.empty(cap * n, dtype=torch.float64, device="cuda")
    out = {}

    def qb():
        out["f"] = eng.device_qb_blocked(A.data_ptr(), m, n, m, False, b, M, tol, 1, 1, R.Omega.philox(12345),
                                         Q.data_ptr(), m, B.data_ptr(), cap, cap)

    tq = timed(qb, 1)
    qb_ph = phases(qb)
    ell = out["f"]["ell"]
    U = torch.empty(m * ell, dtype=torch.float64, device="cuda")
    V = torch.empty(n * ell, dtype=torch.float64, device="cuda")
    S = torch.empty(ell, dtype=torch.float64, device="cuda")
    def svd():
        eng.device_svd_from_qb(Q.data_ptr(), m, m, B.data_ptr(), n, cap, ell, 0, 0, U.data_ptr(), m, S.data_ptr(),
                               V.data_ptr(), n)

    ts = timed(svd, 1)
    ph = phases(svd)
    s = S.cpu().numpy()
    stt = st.cpu().numpy()
    return dict(config="C2", entry="qb_blocked(b=100,M=80,tol=1e-6,q=1) + svd_from_qb(k=0)", m=m, n=n,
                ell=ell, blocks=len(out["f"]["history"]), final_residual=out["f"]["final_residual"],
                tolerance_reached=out["f"]["tolerance_reached"], qb_time_s=tq, svd_time_s=ts, time_s=tq + ts, qb_phases_ms=qb_ph, svd_phases_ms=ph,
                sigma_top100_rel_vs_true=float(np.max(np.abs(s[:100] - stt[:100]) / stt[:100])))


def c3():
    m, n, k, p, q = 20000, 10000, 600, 10, 2
    sig = 10.0 ** (-8.0 * np.arange(1500) / 1500)
    A, st = gen_test_matrix_device(eng, m, n, sig, seed=3, noise=1e-10)
    l = k + p
    jc = torch.empty(n, dtype=torch.int32, device="cuda")
    V = torch.empty(n * k, dtype=torch.float64, device="cuda")
    res = {}

    def run():
        res["r"] = eng.device_id_rand(A.data_ptr(), m, n, m, k, p, q, 1, R.Omega.philox(12345), jc.data_ptr(),
                                      V.data_ptr(), n)

    t = timed(run, 3)
    ph = phases(run)
    F = 2.0 * m * n * l * (2 * q + 1)
    # CUR on device buffers, then through the public host API (+ the 1.6 GB upload)
    dev = {"jc": torch.empty(n, dtype=torch.int32, device="cuda"), "jr": torch.empty(m, dtype=torch.int32, device="cuda"),
           "v": torch.empty(n * k, dtype=torch.float64, device="cuda"), "w": torch.empty(m * k, dtype=torch.float64, device="cuda"),
           "c": torch.empty(m * k, dtype=torch.float64, device="cuda"), "u": torch.empty(k * k, dtype=torch.float64, device="cuda"),
           "r": torch.empty(k * n, dtype=torch.float64, device="cuda")}
    ptrs = {key: t.data_ptr() for key, t in dev.items()}
    tcur = timed(lambda: eng.device_cur_rand(A.data_ptr(), m, n, m, k, p, q, 1, R.Omega.philox(12345), ptrs), 3)
    a_h = A.view(n, m).t().cpu().numpy()
    t0 = time.perf_counter()
    cur = eng.cur_rand(np.asfortranarray(a_h), k, p, q, 1, omega=R.Omega.philox(12345))
    tc = time.perf_counter() - t0
    return dict(config="C3", entry="id_rand + cur_rand", m=m, n=n, k=k, p=p, q=q, id_time_s=t,
                id_tflops=F / t / 1e12, id_qr_residual=res["r"]["qr_residual"], cur_time_s=tcur,
                cur_wall_s_host_api=tc,
                cur_residual=cur["residual"], time_s=t, id_phases_ms=ph)


CONFIGS = {
    "C1": lambda: rsvd_cfg("C1", 2000, 4000, 200, 10, 2, np.exp(-np.arange(2000) / 20.0), seed=1, reps=5),
    "C2": c2,
    "C3": c3,
    "C4": lambda: rsvd_cfg("C4", 50000, 50000, 1000, 20, 4, 1.0 / np.sqrt(np.arange(4000) + 1.0), noise=1e-3,
                           seed=4, reps=2),
    "C5": lambda: rsvd_cfg("C5", 200000, 20000, 500, 10, 2, np.exp(-np.arange(3685) / 100.0), seed=5, reps=3),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CONFIGS)
    for nm in names:
        r = CONFIGS[nm]()
        print(json.dumps(r), flush=True)
        torch.cuda.empty_cache()
