"""CPU-side checks of the C-ABI boundary (no compute calls need a GPU here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, rel_err


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "sgpx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sgpx_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1410_4984_b200 import _lib

    lib = _lib.load()
    declared = _declared_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} missing a ctypes signature"
    assert lib.sgpx_abi_version() == 2


def test_no_cpu_fallback_without_device():
    from paper_1410_4984_b200 import _lib, sgp

    if _lib.load().sgpx_device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(_lib.SgpxCudaError, match="no CPU fallback"):
        sgp.Context(0)


def test_packed_layout_counts():
    from paper_1410_4984_b200 import _lib, sgp

    lib = _lib.load()
    assert lib.sgpx_packed_stats_count(100, 50) == 4 + 5050 + 5000 == sgp.packed_stats_count(100, 50)
    assert lib.sgpx_packed_grads_count(100, 10) == 1 + 10 + 1000 == sgp.packed_grads_count(100, 10)


def test_make_partition_matches_reference(orc):
    from paper_1410_4984_b200 import sgp

    for n, p in [(10, 1), (10, 3), (64000, 32), (1000003, 8)]:
        assert sgp.make_partition(n, p) == orc.make_partition(n, p)
    with pytest.raises(ValueError):
        sgp.make_partition(3, 4)


def _problem(seed=0, n=200, q=3, d=4, m=7):
    rng = np.random.default_rng(seed)
    mu = rng.normal(size=(n, q))
    s = rng.uniform(0.25, 1.0, (n, q))
    y = rng.normal(size=(n, d))
    z = mu[rng.choice(n, m, replace=False)]
    ls = rng.uniform(0.5, 2.0, q)
    return mu, s, y, z, 1.3, ls, 25.0


@pytest.mark.parametrize("latent", [True, False])
def test_coordinator_matches_oracle(orc, latent):
    """The product's fp64 host coordinator (bound_core + adjoints + kern_grads) vs the oracle engine."""
    from paper_1410_4984_b200 import sgp

    mu, s, y, z, var, ls, beta = _problem()
    n, d = y.shape
    ref = orc.engine_evaluate(latent, mu, s, y, z, var, ls, beta, workers=1)
    # statistics from the oracle, KL as the Worker computes it
    st, _ = orc.sweep_stats(latent, mu, s if latent else None, y, z, var, ls)
    kl = 0.5 * np.sum(s + mu ** 2 - np.log(s) - 1.0) if latent else 0.0
    packed = sgp.pack_stats(st.phi, st.yy, n, kl, st.phi_big, st.psi_y)
    k = sgp.KernelSpec(var, ls)
    co = sgp.coordinate_host(1 if latent else 0, n, d, packed, z, k, beta)
    for f in sgp.BOUND_FIELDS:
        assert rel_err(getattr(co["bound"], f), ref.bound[f]) < 1e-10, f
    assert rel_err(co["d_beta"], ref.d_beta) < 1e-10
    # the gradient pass on the oracle with the product's adjoints, then the product's finish
    _, g = orc.sweep_stats(latent, mu, s if latent else None, y, z, var, ls,
                           adj=(co["d_phi"], co["d_psi_y"], co["d_phi_big"]))
    packed_g = np.concatenate([[g.d_variance], g.d_lengthscales, g.d_z.ravel(order="F")])
    dz, dv, dls = sgp.finish_host(packed_g, z, k, co["d_kmm"], co["jitter_factor"])
    assert rel_err(dz, ref.d_z) < 1e-10
    assert rel_err(dv, ref.d_variance) < 1e-10
    assert rel_err(dls, ref.d_lengthscales) < 1e-10


def test_coordinator_errors(orc):
    from paper_1410_4984_b200 import sgp

    mu, s, y, z, var, ls, beta = _problem()
    n, d = y.shape
    st, _ = orc.sweep_stats(True, mu, s, y, z, var, ls)
    packed = sgp.pack_stats(st.phi, st.yy, n, 0.0, st.phi_big, st.psi_y)
    with pytest.raises(ValueError, match="beta must be positive"):
        sgp.coordinate_host(1, n, d, packed, z, sgp.KernelSpec(var, ls), -1.0)
    with pytest.raises(ValueError, match="n_count"):
        sgp.coordinate_host(1, n + 1, d, packed, z, sgp.KernelSpec(var, ls), beta)
    with pytest.raises(ValueError, match="lengthscales must be positive"):
        sgp.coordinate_host(1, n, d, packed, z, sgp.KernelSpec(var, -ls), beta)
