"""Summarise an ncu launch list of tools/profile_step.py into
profiles/rNN_step_kernels.json: the last N launches (one C5 rsvd_v2 call,
N = the "launches_last_call" that profile_step.py printed), grouped by kernel,
with time share, DMMA-pipe activity and DRAM traffic.
Usage: python tools/step_kernels.py LAUNCHES.csv N OUT.json"""
import csv
import re
import json
import sys
from collections import OrderedDict

ROLES = [
    ("dgemm_tma_kernel<0, 1, 0, 1>", "TMA GEMM, A^T*Y power + projection (TN, split-K partials)"),
    ("dgemm_tma_kernel<1, 0, 0, 1>", "TMA GEMM, A*Omega sketch, A*Z power, Y*R^-1, lift (NN)"),
    ("dgemm_tma_kernel<1, 0, 1, 2>", "TMA GEMM sketch with in-register Philox Omega (RLRA_SKETCH_FUSED=1)"),
    ("bgram_jacobi_kernel", "Gram block Jacobi SVD of R-hat (owners + V helpers)"),
    ("cgram_jacobi_kernel", "cluster-resident Gram block Jacobi SVD of R-hat (l <= 256)"),
    ("sgram_jacobi_kernel", "streaming Gram block Jacobi SVD (dynamic visits)"),
    ("dgemm_ws_kernel", "cp.async GEMM (64x64 tiles for short-k / small Grams)"),
    ("dgemm_kernel", "cp.async GEMM (64x64 tiles for short-k / small Grams)"),
    ("block_jacobi_kernel", "one-sided block Jacobi SVD of R-hat"),
    ("chol_inv_coop_kernel", "one-launch Cholesky + R^-1 of the l x l Grams"),
    ("philox_fill_kernel", "Philox Omega materialised for the sketch"),
    ("split_reduce_kernel", "split-K partial reduction"),
    ("tail_reduce_kernel", "tail-wave split-K reduction"),
]


def main(path, n_last, out):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h = rows[0]
    iid, iname, imet, ival = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    launches = OrderedDict()
    for r in rows[1:]:
        d = launches.setdefault(int(r[iid]), {"name": r[iname]})
        d[r[imet]] = float(r[ival].replace(",", ""))
    last = list(launches.values())[-n_last:]
    total_ns = sum(x["gpu__time_duration.sum"] for x in last)
    groups = OrderedDict()
    for x in last:
        key = re.sub(r"^void |rlra_b200::|<?unnamed>::", "", x["name"].split("(")[0])
        g = groups.setdefault(key, {"launches": 0, "ns": 0.0, "dmma_w": 0.0, "dram": 0.0})
        ns = x["gpu__time_duration.sum"]
        g["launches"] += 1
        g["ns"] += ns
        g["dmma_w"] += ns * x.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
        g["dram"] += x.get("dram__bytes_read.sum", 0.0) + x.get("dram__bytes_write.sum", 0.0)
    kernels = []
    for key, g in sorted(groups.items(), key=lambda kv: -kv[1]["ns"]):
        role = next((r for s, r in ROLES if s in key), "")
        kernels.append({"kernel": key, "role": role, "launches": g["launches"], "ms": round(g["ns"] / 1e6, 3),
                        "share": round(g["ns"] / total_ns, 4),
                        "dmma_pipe_pct_of_elapsed": round(g["dmma_w"] / g["ns"], 1),
                        "hbm_gbs": round(g["dram"] / g["ns"], 1), "dram_gb": round(g["dram"] / 1e9, 3)})
    doc = {"source": f"ncu --metrics (cold-cache, serialised) of the last of two C5 rsvd_v2 calls in "
                     f"tools/profile_step.py, {n_last} launches; --clock-control none",
           "total_ms": round(total_ns / 1e6, 2), "kernels": kernels}
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps({k["kernel"]: (k["ms"], k["share"]) for k in kernels[:6]}))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3])
