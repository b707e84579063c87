"""GPU test-matrix generator (reference testmat.hpp:65-74).

A = U diag(sigma) V^T (+ noise * G) built on the device by the engine
(rlra_gen_test_matrix: Philox Gaussians, CholQR2 orthonormalisation, the DMMA
GEMM).  The
reference builds U and V with a Householder QR on the CPU, which is
infeasible at C4/C5 sizes (a 200000 x 20000 QR); the spectrum, not the
particular U and V, is what the configs specify.  torch only allocates.
"""
from __future__ import annotations

import numpy as np


def gen_test_matrix_device(eng, m: int, n: int, sigma, seed: int, noise: float = 0.0,
                           noise_seed: int | None = None):
    """Return (A, sigma) with A a flat torch float64 CUDA tensor holding the
    m x n matrix column-major (ld = m) and sigma the r singular values used.
    The generator is the engine's (rlra_gen_test_matrix, csrc/io.cu)."""
    import torch

    dev = torch.device("cuda", eng.device)
    sigma = np.asarray(sigma, dtype=np.float64)
    if len(sigma) > min(m, n):
        raise ValueError("spectrum longer than min(m, n)")
    if noise_seed is not None and noise_seed != seed:
        raise ValueError("the noise draw is keyed by the matrix seed")
    A = torch.empty(m * n, dtype=torch.float64, device=dev)
    eng.device_gen_test_matrix(m, n, sigma, seed, noise, A.data_ptr(), m)
    return A, torch.as_tensor(sigma, device=dev)
