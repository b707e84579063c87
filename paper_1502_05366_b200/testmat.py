"""GPU test-matrix generator (reference testmat.hpp:65-74).

A = U diag(sigma) V^T (+ noise * G) built on the device with the engine's own
kernels: Philox Gaussians, CholQR2 orthonormalisation, the DMMA GEMM.  The
reference builds U and V with a Householder QR on the CPU, which is
infeasible at C4/C5 sizes (a 200000 x 20000 QR); the spectrum, not the
particular U and V, is what the configs specify.  torch only allocates.
"""
from __future__ import annotations

import numpy as np


def gen_test_matrix_device(eng, m: int, n: int, sigma, seed: int, noise: float = 0.0,
                           noise_seed: int | None = None):
    """Return (A, sigma) with A a flat torch float64 CUDA tensor holding the
    m x n matrix column-major (ld = m) and sigma the r singular values used."""
    import torch

    dev = torch.device("cuda", eng.device)
    sigma = np.asarray(sigma, dtype=np.float64)
    r = len(sigma)
    if r > min(m, n):
        raise ValueError("spectrum longer than min(m, n)")
    U = torch.empty(r * m, dtype=torch.float64, device=dev)
    V = torch.empty(r * n, dtype=torch.float64, device=dev)
    eng.device_gaussian_philox(m, r, seed, 101, 0, U.data_ptr(), m)
    eng.device_gaussian_philox(n, r, seed, 102, 0, V.data_ptr(), n)
    eng.device_orth(U.data_ptr(), m, r)
    eng.device_orth(V.data_ptr(), n, r)
    s = torch.as_tensor(sigma, device=dev)
    U.view(r, m).mul_(s.view(r, 1))  # scale column j of U by sigma_j
    A = torch.empty(m * n, dtype=torch.float64, device=dev)
    eng.device_matmul(False, True, U.data_ptr(), m, r, m, V.data_ptr(), n, r, n, A.data_ptr(), m)
    eng.synchronize()
    del U, V
    if noise:
        G = torch.empty(m * n, dtype=torch.float64, device=dev)
        eng.device_gaussian_philox(m, n, seed if noise_seed is None else noise_seed, 103, 0,
                                   G.data_ptr(), m)
        A.add_(G, alpha=noise)
        torch.cuda.synchronize(dev)
        del G
    return A, s
