"""Synthetic workloads of the benchmark configurations, from the reference's
own generator so the GPU engine and the CPU reference see identical inputs.

Latent (Bayesian GP-LVM, C2 / C3 / C5): mu = Rng(seed).normal_matrix(N, Q), S = 0.5 (the init_gplvm
default, model.hpp:431), Y = Rng(seed + 1).normal_matrix(N, D), Z = the M rows of mu init_gplvm would
pick with Rng(seed + 2) (model.hpp:420-429); variance = lengthscales = 1, beta = 100.
Regression (SGPR, C1 / C4): X = Rng(seed).normal_matrix(N, Q), Y = Rng(seed + 1).normal_matrix(N, D),
Z = M rows of X as above; variance = lengthscales = beta = 1 (bench.hpp:157-160).
The normals are generated on the GPU (sgpx_rng_normal_matrix) when ``device`` is given.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import sgp


@dataclass
class Workload:
    latent: bool
    mu: object        # N x Q (X for regression): numpy (Fortran) or column-major CUDA tensor
    s: object         # N x Q or None
    y: object         # N x D
    z: np.ndarray     # M x Q (host)
    variance: float
    lengthscales: np.ndarray
    beta: float

    @property
    def kernel(self) -> sgp.KernelSpec:
        return sgp.KernelSpec(self.variance, self.lengthscales)


def make(latent: bool, n: int, q: int, d: int, m: int, seed: int = 0, device=None, s_value: float = 0.5,
         ctx=None) -> Workload:
    mu = sgp.rng_normal_matrix(seed, n, q, device=device, ctx=ctx)
    y = sgp.rng_normal_matrix(seed + 1, n, d, device=device, ctx=ctx)
    idx = sgp.rng_choose_rows(seed + 2, n, m)
    if device is not None:
        import torch

        z = np.asfortranarray(mu[torch.as_tensor(idx, device=mu.device)].cpu().numpy())
        s = torch.full((q, n), s_value, dtype=torch.float64, device=device).t() if latent else None
    else:
        z = np.asfortranarray(mu[idx])
        s = np.full((n, q), s_value, order="F") if latent else None
    beta = 100.0 if latent else 1.0
    return Workload(latent, mu, s, y, z, 1.0, np.ones(q), beta)
