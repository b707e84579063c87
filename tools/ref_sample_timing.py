"""Time the UNMODIFIED reference (oracle/_ref/librlra_ref_fast.so, all host
threads) on proportional samples of C5: (m, n, l) scaled by 1/S with p = 10
and q = 2 kept, so every phase keeps its share of the work (GEMM ~ m n l,
the serial Householder orths ~ (m + n) l^2).  Compared with the one-off full
C5 run (profiles/r02_parity_full.jsonl: 1139 s = 21.5 GFLOP/s on 16 threads)
it picks the bench reference arm's sample.  Prints one JSON line per run."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import _oracle

ref = _oracle._Lib(_oracle.REF_FAST_PATH, "ref_")
cores = os.cpu_count() or 1
ref.lib.ref_set_threads(cores)
for S in [int(x) for x in (sys.argv[1:] or ["4", "5", "8"])]:
    m, n, l = 200000 // S, 20000 // S, 510 // S
    k, p, q = l - 10, 10, 2
    rs = np.random.default_rng(5)
    a = np.asfortranarray(rs.standard_normal((m, n)))
    for rep in range(2):
        t0 = time.perf_counter()
        ref.rsvd(a, k, p, q, 1, ref.rng(12345), 0)
        dt = time.perf_counter() - t0
        fl = 4.0 * m * n * (k + p) * (q + 1)
        print(json.dumps(dict(scale=S, m=m, n=n, k=k, p=p, q=q, seconds=dt, gflops=fl / dt / 1e9, threads=cores,
                              rep=rep)), flush=True)
