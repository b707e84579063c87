#!/usr/bin/env python
"""bench.py — headline benchmark: rsvd_v2 on the C5 configuration.

Workload (BASELINE.json configs[4], the north_star target and the config
scaled at 1/2/4/8 GPUs): A = U diag(s) V^T, m=200000, n=20000 (32 GB FP64),
s_j = exp(-j/100) (truncated at the 3685 modes above 1e-16),
U, V orthonormalised seeded Gaussians; k=500, p=10, q=2, s=1.  One step is
one full rlra_rsvd(v2) call (sketch, 2 power iterations with CholQR2
re-orthonormalisation, projection, QR of B^T, Jacobi SVD of R, lift).

metric  : effective FP64 TFLOP/s = F_gemm / step time with
          F_gemm = 4 m n l (q+1) (2.448e13 flop for C5);
value   : A resident in HBM, Omega drawn from Philox inside the call
          (materialised once, n x l, then the streaming GEMM);
e2e     : the same call through the C-ABI with HOST buffers (pinned A in,
          U/sigma/V out), host<->device copies inside the timed region; the
          engine streams the 32 GB upload in row chunks on a copy stream
          under the sketch GEMM (engine.cu upload_and_sketch);
roofline: the dominant kernel is the FP64 DMMA GEMM; achieved = its
          algorithmic flops / its CUDA-event time on the engine stream over
          the timed region, against the measured DMMA peak
          (tools/fp64_peak.cu: 37.1 TFLOP/s; MEASURED_PEAKS.json has no FP64
          entry).
A (32 GB) is far larger than L2 (126 MB), so no flush is needed between steps.

--impl reference: the reference's own CPU implementation (oracle/_ref, the
unmodified headers) on a proportional 1/5 sample of the same workload (m, n
and k + p scaled, see CPU_SCALE), all host cores, --warmup/--steps honoured.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_DMMA_PEAK_TFLOPS = 37.1  # tools/fp64_peak.cu on this pool's B200 (DMMA.8x8x4, 1965 MHz)
C5 = dict(m=200000, n=20000, k=500, p=10, q=2, s=1)
SEED_GEN = 5          # generator seed = config number
SEED_OMEGA = 12345    # CLI default seed (rlra_cli.cpp:56)
CPU_SAMPLE = dict(m=600, n=4000)  # bounded row/column slice of C5 for the CPU legs


def f_gemm(m, n, k, p, q, **_):
    return 4.0 * m * n * (k + p) * (q + 1)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def self_launch(n, share_gpus=False):
    """--gpus N without a launcher: start N ranks of this script (one process
    per GPU, the environment torch.distributed.run would set) and wait; rank
    0's stdout is the JSON line."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < n and not share_gpus:  # (--comm host lets ranks share GPUs)
        print(f"bench.py: --gpus {n} but only {have} GPU(s) visible", file=sys.stderr)
        return 1
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    rcs = [p.wait() for p in procs]
    return max(rcs, key=abs)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# The CPU legs time a PROPORTIONAL sample of C5: m, n and l = k + p scaled by
# 1/5 (p = 10, q = 2 kept), so every phase keeps its share of the work (the
# threaded GEMMs ~ m n l, the reference's serial Householder orths ~ (m + n)
# l^2) and one reference rsvd takes ~8 s on the box's 16 threads.  A
# full-width slab (m' x 20000, k = 500) cannot fit the driver's budget: its
# n-side serial orths and QR of B^T alone take ~40 s per step.  Measured on the
# box (tools/ref_sample_timing.py, profiles/r02_ref_sample_timing.jsonl): 23.5-
# 24.9 GFLOP/s at scales 1/4, 1/5 and 1/8 against 21.5 GFLOP/s for the one-off
# full C5 reference run (1139 s, profiles/r02_parity_full.jsonl), so the sample
# rate is within ~13 % of the full-size rate (slightly flattering the CPU).
CPU_SCALE = 5
CPU_SAMPLE = dict(m=C5["m"] // CPU_SCALE, n=C5["n"] // CPU_SCALE, k=(C5["k"] + C5["p"]) // CPU_SCALE - C5["p"],
                  p=C5["p"], q=C5["q"], s=C5["s"])
FULL_C5_REFERENCE_S = 1138.98  # profiles/r02_parity_full.jsonl: unmodified reference, 16 threads, same A


def cpu_reference_step(a_sample, cores):
    """One rsvd_v2 on the reference CPU build (all `cores` threads); seconds."""
    import ctypes as C

    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import _oracle

    lib = C.CDLL(_oracle.REF_FAST_PATH)
    lib.ref_set_threads(cores)
    m, n = a_sample.shape
    k, p, q, s = CPU_SAMPLE["k"], CPU_SAMPLE["p"], CPU_SAMPLE["q"], CPU_SAMPLE["s"]
    r = _oracle.Rng()
    lib.ref_rng_seed(C.byref(r), C.c_uint64(SEED_OMEGA))
    u = np.zeros((m, k), order="F")
    sg = np.zeros(k)
    v = np.zeros((n, k), order="F")
    t0 = time.perf_counter()
    st = lib.ref_rsvd(0, _oracle.d(a_sample), m, n, k, p, q, s, C.byref(r), _oracle.d(u),
                      _oracle.d(sg), _oracle.d(v))
    dt = time.perf_counter() - t0
    if st != 0:
        raise RuntimeError("reference rsvd failed")
    return dt


def cpu_port_step(a_sample):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import _oracle

    o = _oracle.orc()
    t0 = time.perf_counter()
    o.rsvd(a_sample, CPU_SAMPLE["k"], CPU_SAMPLE["p"], CPU_SAMPLE["q"], CPU_SAMPLE["s"], o.rng(SEED_OMEGA), 0)
    return time.perf_counter() - t0


def cpu_sample_matrix():
    """The proportional CPU sample of C5: a (m/5) x (n/5) matrix U diag(s) V^T
    with the C5 law in the scaled index (s_j = exp(-5 j / 100), 737 modes),
    U, V orthonormalised seeded Gaussians (numpy)."""
    import numpy as np

    m, n = CPU_SAMPLE["m"], CPU_SAMPLE["n"]
    rs = np.random.default_rng(SEED_GEN)
    r = 3685 // CPU_SCALE
    U, _ = np.linalg.qr(rs.standard_normal((m, r)))
    V, _ = np.linalg.qr(rs.standard_normal((n, r)))
    s = np.exp(-CPU_SCALE * np.arange(r) / 100.0)
    return np.asfortranarray((U * s) @ V.T)


def cpu_sample_desc():
    c = CPU_SAMPLE
    return (f"rsvd_v2 on a proportional C5 sample: m, n, k+p scaled 1/{CPU_SCALE} "
            f"({c['m']}x{c['n']}, k={c['k']}, p={c['p']}, q={c['q']}); the full C5 reference run took "
            f"{FULL_C5_REFERENCE_S:.0f} s = {f_gemm(**C5) / FULL_C5_REFERENCE_S / 1e12:.4f} TFLOP/s on 16 threads")


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import _oracle

    a = cpu_sample_matrix()
    cores = os.cpu_count() or 1
    use_ref = os.path.exists(_oracle.REF_FAST_PATH)
    fl = f_gemm(**CPU_SAMPLE)
    for _ in range(args.warmup):
        cpu_reference_step(a, cores) if use_ref else cpu_port_step(a)
    total = 0.0
    for _ in range(args.steps):
        total += cpu_reference_step(a, cores) if use_ref else cpu_port_step(a)
    t = total / args.steps
    val = fl / t / 1e12
    c = CPU_SAMPLE
    line = {
        "impl": "reference",
        "metric": "rsvd_v2 effective FP64 TFLOP/s (F_gemm = 4mnl(q+1) / time), C5 workload",
        "value": val, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C5 rsvd_v2 (m=200000,n=20000,k=500,p=10,q=2); CPU proportional sample "
                               f"1/{CPU_SCALE}: m={c['m']} n={c['n']} k={c['k']} p={c['p']} q={c['q']}",
                   "sample_m": c["m"], "sample_n": c["n"], "sample_k": c["k"],
                   "full_c5_reference_s": FULL_C5_REFERENCE_S,
                   "full_c5_reference_tflops": f_gemm(**C5) / FULL_C5_REFERENCE_S / 1e12},
        "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": cores if use_ref else 1,
                         "kind": "reference" if use_ref else "port", "sample": cpu_sample_desc()},
        "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def generate_c5(eng, torch, dev, m, n, seed):
    """A = U diag(s) V^T on the device with the engine's own kernels:
    Philox Gaussians, CholQR2 orthonormalisation, DMMA GEMM (the GPU
    generator of SURVEY.md §8f row 1; testmat.hpp:65-74 semantics)."""
    import paper_1502_05366_b200 as R

    r = 3685  # modes with exp(-j/100) > 1e-16
    U = torch.empty(r * m, dtype=torch.float64, device=dev)
    V = torch.empty(r * n, dtype=torch.float64, device=dev)
    eng.device_gaussian_philox(m, r, seed, 101, 0, U.data_ptr(), m)
    eng.device_gaussian_philox(n, r, seed, 102, 0, V.data_ptr(), n)
    eng.device_orth(U.data_ptr(), m, r)
    eng.device_orth(V.data_ptr(), n, r)
    s = torch.exp(-torch.arange(r, dtype=torch.float64, device=dev) / 100.0)
    U.view(r, m).mul_(s.view(r, 1))  # column j of U (col-major) scaled by s_j
    A = torch.empty(m * n, dtype=torch.float64, device=dev)
    eng.device_matmul(False, True, U.data_ptr(), m, r, m, V.data_ptr(), n, r, n, A.data_ptr(), m)
    eng.synchronize()
    del U, V
    return A, s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--m", type=int, default=C5["m"])
    ap.add_argument("--n", type=int, default=C5["n"])
    ap.add_argument("--dist", action="store_true",
                    help="use the row-sharded NCCL path even at N=1 (exercises dist.py)")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "host"],
                    help="host: the drivers' host-staged collectives over gloo with a GPU token, so "
                         "ranks may share a GPU (functional test of the N-rank path; not a timing)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args.gpus, share_gpus=args.comm == "host"))

    import numpy as np
    import torch

    import paper_1502_05366_b200 as R

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} ranks")
    if args.comm == "host":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    use_dist = world > 1 or args.dist
    if use_dist:
        import torch.distributed as dist
        # the driver reads nranks from NCCL's INIT lines; the algorithm and
        # protocol are pinned so the row sums (and every replicated factor)
        # are reproducible run to run (csrc/dist.cu pin_nccl_env)
        if world > 1:
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        # NCCL's log lines (INIT info, its version banner) go to stderr: stdout
        # carries only the JSON line
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        os.environ.setdefault("NCCL_ALGO", "Ring")
        os.environ.setdefault("NCCL_PROTO", "Simple")
        if world > 1:
            if args.comm == "host":
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=dev)
        else:  # --dist at N=1: exercise the row-sharded path with a 1-rank NCCL group
            import socket
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
            sk.close()
            dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                    world_size=1, device_id=dev)
    eng = R.Engine(local)
    cfg = dict(C5)
    cfg["m"], cfg["n"] = args.m, args.n
    m, n, k, p, q, s = cfg["m"], cfg["n"], cfg["k"], cfg["p"], cfg["q"], cfg["s"]
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)
    if not use_dist:
        # one GPU: the whole factorization is one C-ABI call
        m_loc, row0 = m, 0
        A, sig_true = generate_c5(eng, torch, dev, m, n, SEED_GEN)
        U = torch.empty(m * k, dtype=torch.float64, device=dev)
        V = torch.empty(n * k, dtype=torch.float64, device=dev)
        S = torch.empty(k, dtype=torch.float64, device=dev)

        def step(seed):
            eng.device_rsvd(R.RSVD_V2, A.data_ptr(), m, n, m, k, p, q, s, R.Omega.philox(seed),
                            U.data_ptr(), S.data_ptr(), V.data_ptr())
    else:
        # N GPUs: A row-sharded (strong scaling of the same C5 matrix), NCCL
        # allreduce of the Grams and of the n x l partials (dist.py)
        from paper_1502_05366_b200 import dist as D

        # the C++ driver's own NCCL communicator (or, --comm host, its
        # host-staged collectives over the gloo group with a GPU token)
        comm = D.HostComm(eng, share_gpu=True) if args.comm == "host" else D.NcclComm(eng)
        bounds = np.linspace(0, m, world + 1).astype(int)
        row0, m_loc = int(bounds[rank]), int(bounds[rank + 1] - bounds[rank])
        Ad, sig_true = D.gen_test_matrix_rowsharded(comm, n, row0, m_loc, m,
                                                    np.exp(-np.arange(3685) / 100.0), SEED_GEN)
        A = Ad.t
        out = {}

        def step(seed):  # csrc/dist.cu through rlra_rsvd_rowsharded
            out["U"], out["S"], out["V"] = D.rsvd_v2_native(comm, Ad, m, k, p, q, s, R.Omega.philox(seed))

    for w in range(args.warmup):
        step(SEED_OMEGA + w)
    eng.synchronize()
    if use_dist:
        torch.distributed.barrier()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    eng.profile(True)
    launches0 = eng.launches
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for i in range(args.steps):
        step(SEED_OMEGA + 100 + i)
    ev1.record(stream)
    ev1.synchronize()
    launches = eng.launches - launches0
    prof = eng.profile_records()
    eng.profile(False)
    clk = clocks.stop()
    ms_total = ev0.elapsed_time(ev1)
    rdev = dev if (use_dist and args.comm == "nccl") else torch.device("cpu")  # collective tensors
    if use_dist:
        t = torch.tensor([ms_total], device=rdev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    F = f_gemm(m, n, k, p, q)
    value = F / (ms_step * 1e-3) / 1e12  # the whole job: one C5 factorization per step

    # dominant kernel: the DMMA GEMMs that stream A (M or K == m)
    big = [r for r in prof if r["name"] in ("gemm_sketch", "gemm_power", "gemm_proj")]
    g_ms = sum(r["ms"] for r in big)
    g_fl = sum(r["flops"] for r in big)
    # phases are nested intervals: orth contains chol and gemm_orth, chol contains gemm_chol
    phases = {}
    for r in prof:
        phases[r["name"]] = phases.get(r["name"], 0.0) + r["ms"] / args.steps
    sweeps = [r["K"] for r in prof if r["name"] == "small_svd"]
    if sweeps:
        phases["small_svd_sweeps"] = sweeps[-1]
    achieved = g_fl / (g_ms * 1e-3) / 1e12 if g_ms > 0 else None

    # relative error of the last factorization (device reduction)
    if not use_dist:
        err = eng.device_rel_error(A.data_ptr(), m, n, U.data_ptr(), S.data_ptr(), V.data_ptr(), k)
    else:
        U, S, V = out["U"].t, out["S"].t[:k], out["V"].t
        e_loc = eng.device_rel_error(A.data_ptr(), m_loc, n, U.data_ptr(), S.data_ptr(), V.data_ptr(), k)
        a2 = float(torch.sum(A ** 2))
        tt = torch.tensor([e_loc ** 2 * a2, a2], dtype=torch.float64, device=rdev)
        torch.distributed.all_reduce(tt)
        err = float(torch.sqrt(tt[0] / tt[1]))
    sig = S.cpu().numpy()
    st = sig_true[:k].cpu().numpy()
    sig_rel = float(np.max(np.abs(sig[:100] - st[:100]) / st[:100]))

    line = {
        "metric": "rsvd_v2 effective FP64 TFLOP/s (F_gemm = 4mnl(q+1) / time), C5 workload",
        "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: A = U diag(exp(-j/100)) V^T, U,V orthonormalised Philox Gaussians "
                "(3685 modes), generated on the GPU",
        "config": {"workload": f"C5 rsvd_v2 m={m} n={n} k={k} p={p} q={q} s={s}",
                   "omega": "philox (materialised per call, n x l)", "l2": "A (32 GB) >> L2; no flush needed",
                   "parallelism": "1 GPU" if not use_dist else
                   f"A row-sharded over {world} GPUs ({m_loc} rows/rank), C++ driver "
                   "(rlra_rsvd_rowsharded) with NCCL allreduce of Grams and n x l partials"
                   if args.comm == "nccl" else
                   f"FUNCTIONAL TEST, not a timing: {world} ranks sharing GPUs through host-staged "
                   "collectives over gloo with a GPU token (rlra_comm_create_host)"},
        "time_s": ms_step / 1e3,
        "frac_of_fp64_peak": value / world / FP64_DMMA_PEAK_TFLOPS,
        "phases_ms": {k_: round(v_, 3) for k_, v_ in sorted(phases.items())},
        "rel_error": {"fro": err, "sigma_top100_vs_true_max_rel": sig_rel},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": FP64_DMMA_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": (achieved / FP64_DMMA_PEAK_TFLOPS) if achieved else None,
                     # dram__bytes_read.sum + write.sum of the dominant launch (the TN
                     # A^T*Y product) in one ncu --set full capture
                     # (profiles/r02_gemm_tma_ncu_summary.md): 36.15 GB read + 0.32 GB
                     # write vs 32.0 GB algorithmic (A read once)
                     "traffic": 36.146e9 + 0.3207e9,
                     "traffic_unit": "bytes/launch (TN A^T*Y GEMM)",
                     "kernel": "dgemm_tma_kernel (A-streaming products: sketch, 2q power, projection)",
                     "peak_source": "measured DMMA peak, tools/fp64_peak.cu (MEASURED_PEAKS.json has no FP64 entry)"},
        "gpu_launches": launches,
        "clocks": clk,
    }

    # ---------------------------------------------- e2e through the C-ABI --
    if not args.no_e2e:
        Ah = torch.empty(m_loc * n, dtype=torch.float64, pin_memory=True)
        Ah.copy_(A)
        Uh = torch.empty(m_loc * k, dtype=torch.float64, pin_memory=True)
        Vh = torch.empty(n * k, dtype=torch.float64, pin_memory=True)
        Sh = torch.empty(k, dtype=torch.float64, pin_memory=True)
        e2e_steps = max(1, min(args.steps, 3))
        if not use_dist:
            del A
            torch.cuda.empty_cache()

            def estep(seed):  # the drop-in call with host buffers
                eng.host_rsvd_ptr(R.RSVD_V2, Ah.data_ptr(), m, n, m, k, p, q, s,
                                  R.Omega.philox(seed), Uh.data_ptr(), Sh.data_ptr(), Vh.data_ptr())
            path = "rlra_rsvd(loc=RLRA_HOST), pinned host A, row-chunked upload overlapped with the sketch"
        else:
            del A, Ad
            out.clear()
            torch.cuda.empty_cache()

            def estep(seed):  # each rank's drop-in call with its pinned host shard
                eng.host_rsvd_rowsharded_ptr(comm.handle, Ah.data_ptr(), m_loc, n, m_loc, m, k, p, q, s,
                                             R.Omega.philox(seed), Uh.data_ptr(), m_loc, Sh.data_ptr(),
                                             Vh.data_ptr(), n)
            path = ("rlra_rsvd_rowsharded(loc=RLRA_HOST) per rank, pinned host shard, row-chunked upload "
                    "overlapped with the local sketch")

        estep(SEED_OMEGA)
        if use_dist:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        # CUDA events on the engine stream bracket the calls (each call is
        # synchronous: H2D, compute, D2H all inside); max over the ranks
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(e2e_steps):
            estep(SEED_OMEGA + 200 + i)
        e1.record(stream)
        e1.synchronize()
        te = e0.elapsed_time(e1) * 1e-3 / e2e_steps
        if use_dist:
            tt = torch.tensor([te], dtype=torch.float64, device=rdev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            te = float(tt.item())
        line["e2e"] = {"value": F / te / 1e12, "unit": "TFLOP/s",
                       "h2d_bytes_per_step": 8 * m * n,
                       "d2h_bytes_per_step": 8 * (m * k + world * (n * k + k)),
                       "ms_per_step": te * 1e3, "steps": e2e_steps, "path": path}

    # ------------------------------------------------------ cpu baseline --
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            import _oracle
            a = cpu_sample_matrix()
            cores = os.cpu_count() or 1
            use_ref = os.path.exists(_oracle.REF_FAST_PATH)
            dt = cpu_reference_step(a, cores) if use_ref else cpu_port_step(a)
            line["cpu_baseline"] = {
                "value": f_gemm(**CPU_SAMPLE) / dt / 1e12, "unit": "TFLOP/s", "cores": cores if use_ref else 1,
                "kind": "reference" if use_ref else "port", "sample": cpu_sample_desc() + f"; this step {dt:.2f} s"}
        except Exception as e:  # reported, never silently substituted
            line["cpu_baseline"] = {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "reference",
                                    "sample": f"failed: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if use_dist:
        comm.close()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
