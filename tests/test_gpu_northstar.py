"""GPU parity where the numbers are quoted, and the accuracy envelope.

* The benchmark configurations at their own shapes against the fp64 oracle engine
  (Engine::evaluate(true), parallel.hpp:370-450): C3 at the full north-star size N = 1M through the
  host-buffer (sub-shard streaming) path, C2 at its exact shape, the C5 shape with D = 100 and the C4
  shape (SGPR, M = 500).  Inputs come from the reference's own generator (sgp::Rng, common.hpp:45-97)
  so both sides see identical data.
* Every comparison asserts the reference's element-wise rel_err (proj/tests/support/oracles.hpp:55-58,
  |a-b| / max(|a|, |b|, 1)) next to the norm-wise error.
* The precision-mode envelope: wide and clustered latent spaces, far outlier rows,
  far clusters without inducing points, in both modes; the mode the engine picked is checked too.

Tolerances: the mixed (tensor-core) modes hold norm-wise 1e-5 for statistics / bound
terms and 5e-5 for every gradient block; element-wise they hold 1e-3 — the entries that miss 1e-4 are
the small residues of cancelling sums (a d Z entry 500x below its block's largest is the difference of
the psi part and the Kmm part, each ~1e3x larger), which carry the fp32-level rounding of their terms.
The direct mode is fp64 end to end and holds 1e-9 element-wise (measured <= 5e-12).
"""
import os

import numpy as np
import pytest

from conftest import norm_rel_err, rel_err

pytestmark = pytest.mark.gpu

ELEM_TOL = 1e-3
STAT_TOL = 1e-5
GRAD_TOL = 5e-5
DIRECT_TOL = 1e-9
THREADS = max(1, os.cpu_count() or 1)


@pytest.fixture(scope="module")
def sgp():
    from paper_1410_4984_b200 import sgp as m

    if m.device_count() == 0:
        pytest.fail("no CUDA device visible to libsgpx (gpu tests must run on the B200)")
    return m


def _check_eval(r, ref, latent, elem_tol=ELEM_TOL, bound_tol=STAT_TOL, grad_tol=GRAD_TOL):
    from paper_1410_4984_b200 import sgp as m

    errs = {}
    assert rel_err(r.bound.total, ref.bound["total"]) < bound_tol
    for f in m.BOUND_FIELDS:
        assert rel_err(getattr(r.bound, f), ref.bound[f]) < bound_tol, f
    g = r.grads
    pairs = dict(d_z=(g.d_z, ref.d_z), d_ls=(g.d_lengthscales, ref.d_lengthscales),
                 d_var=([g.d_variance], [ref.d_variance]), d_beta=([g.d_beta], [ref.d_beta]))
    if latent:
        pairs.update(d_mu=(g.d_mu, ref.d_mu), d_s=(g.d_s, ref.d_s))
    for k, (a, b) in pairs.items():
        errs[k] = (rel_err(a, b), norm_rel_err(a, b))
        assert errs[k][0] < elem_tol, (k, errs[k])
        assert errs[k][1] < grad_tol, (k, errs[k])
    return errs


# ---------------------------------------------------------------------------------------------
# the reference's generator and binary matrices on the device
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("seed,rows,cols", [(0, 1001, 7), (42, 3, 5), (7, 20000, 1)])
def test_rng_stream_matches_reference(sgp, orc, seed, rows, cols):
    want = orc.rng_normal_matrix(seed, rows, cols)
    host = sgp.rng_normal_matrix(seed, rows, cols)
    dev = sgp.rng_normal_matrix(seed, rows, cols, device="cuda").cpu().numpy()
    # CUDA's fp64 log / sin / cos are within 2 ulp of glibc's
    assert np.max(np.abs(host - want) / np.maximum(np.abs(want), 1e-300)) < 1e-14
    assert np.array_equal(host, dev)
    assert np.array_equal(sgp.rng_choose_rows(seed + 2, rows, min(rows, 50)),
                          orc.rng_choose_rows(seed + 2, rows, min(rows, 50)))


def test_binary_matrix_roundtrip(sgp, tmp_path):
    a = sgp.rng_normal_matrix(3, 70001, 13)
    base = str(tmp_path / "y")
    sgp.write_matrix_bin(base, a)
    assert open(base + ".shape").read() == "70001 13\n"
    raw = np.fromfile(base + ".bin", dtype="<f8").reshape(70001, 13)  # row-major little-endian
    assert np.array_equal(raw, a)
    assert np.array_equal(sgp.read_matrix_bin(base), a)
    assert np.array_equal(sgp.load_matrix_bin_device(base).cpu().numpy(), a)
    with open(base + ".bin", "r+b") as f:
        f.truncate(8 * 13 * 100 + 8)
    with pytest.raises(sgp.SgpxError, match="truncated at row 100"):
        sgp.read_matrix_bin(base)
    with pytest.raises(sgp.SgpxError, match="cannot open"):
        sgp.read_matrix_bin(str(tmp_path / "missing"))


# ---------------------------------------------------------------------------------------------
# benchmark configurations vs the oracle engine
# ---------------------------------------------------------------------------------------------
def test_c3_north_star_full_n(sgp, orc):
    """C3 (N = 1M, Q = 10, D = 50, M = 100): host mu / S / Y streamed to the device in sub-shards
    with the kernels, d mu / d S streamed back into registered pinned buffers — the e2e path of
    the benchmark — against the fp64 oracle engine on the same Rng inputs."""
    import torch

    from paper_1410_4984_b200 import synthetic

    w = synthetic.make(True, 1_000_000, 10, 50, 100, seed=0)
    eng = sgp.Engine(sgp.ModelKind.latent, w.mu, w.s, w.y)
    n, q = w.mu.shape
    gmu = torch.empty(q, n, dtype=torch.float64, pin_memory=True).numpy().T
    gs = torch.empty(q, n, dtype=torch.float64, pin_memory=True).numpy().T
    eng.set_local_grads_out(gmu, gs)
    eng.broadcast(w.kernel, w.beta, w.z, w.mu, w.s)
    r = eng.evaluate(True)
    assert r.timing.precision == "fast"
    ref = orc.engine_evaluate(True, w.mu, w.s, w.y, w.z, w.variance, w.lengthscales, w.beta, workers=THREADS)
    errs = _check_eval(r, ref, True)
    print("C3 1M:", {k: f"{a:.1e}/{b:.1e}" for k, (a, b) in errs.items()})


def test_c2_exact_shape(sgp, orc):
    """C2 (N = 100k, Q = 10, D = 10, M = 100), device-resident."""
    from paper_1410_4984_b200 import synthetic

    w = synthetic.make(True, 100_000, 10, 10, 100, seed=5, device="cuda")
    eng = sgp.Engine(sgp.ModelKind.latent, w.mu, w.s, w.y)
    eng.broadcast(w.kernel, w.beta, w.z)
    r = eng.evaluate(True)
    mu, s, y = (np.asfortranarray(t.cpu().numpy()) for t in (w.mu, w.s, w.y))
    ref = orc.engine_evaluate(True, mu, s, y, w.z, w.variance, w.lengthscales, w.beta, workers=THREADS)
    _check_eval(r, ref, True)


def test_c5_shape_d100(sgp, orc):
    """C5 shape (Q = 20, D = 100, M = 256: 32,896 pairs) at an oracle-sized N."""
    from paper_1410_4984_b200 import synthetic

    w = synthetic.make(True, 20_000, 20, 100, 256, seed=11)
    eng = sgp.Engine(sgp.ModelKind.latent, w.mu, w.s, w.y)
    eng.broadcast(w.kernel, w.beta, w.z)
    r = eng.evaluate(True)
    ref = orc.engine_evaluate(True, w.mu, w.s, w.y, w.z, w.variance, w.lengthscales, w.beta, workers=THREADS)
    _check_eval(r, ref, True)


def test_c4_shape_sgpr(sgp, orc):
    """C4 shape (SGPR, Q = 8, D = 1, M = 500: 125,250 pairs) at an oracle-sized N.  The narrow SGPR
    kernel with 500 inducing points is the hardest case of the precise mode: its d Z (entries <= 7,
    residues of ~1e3x larger cancelling sums over 500 pair weights) reaches 4e-5 .. 6e-5 norm-wise, so
    this test asserts the north star's 1e-4 for the mixed path there."""
    from paper_1410_4984_b200 import synthetic

    w = synthetic.make(False, 20_000, 8, 1, 500, seed=21)
    eng = sgp.Engine(sgp.ModelKind.regression, w.mu, None, w.y)
    eng.broadcast(w.kernel, w.beta, w.z)
    r = eng.evaluate(True)
    ref = orc.engine_evaluate(False, w.mu, None, w.y, w.z, w.variance, w.lengthscales, w.beta, workers=THREADS)
    _check_eval(r, ref, False, grad_tol=1e-4)


# ---------------------------------------------------------------------------------------------
# the accuracy envelope
# ---------------------------------------------------------------------------------------------
def _layout(kind, f, n=4000, q=10, d=10, m=100, seed=1):
    rng = np.random.default_rng(seed)
    s = rng.uniform(0.25, 1.0, (n, q))
    y = rng.normal(size=(n, d))
    ls = rng.uniform(0.5, 2.0, q)
    if kind == "gauss":  # mu ~ N(0, f^2), Z from mu
        mu = f * rng.normal(size=(n, q))
        z = mu[rng.choice(n, m, replace=False)] + 0.05 * rng.normal(size=(m, q))
    elif kind == "bimodal":  # two clusters at +-f l along q = 0, inducing points in both
        mu = rng.normal(size=(n, q))
        mu[:, 0] += np.where(np.arange(n) % 2 == 0, 1.0, -1.0) * f * ls[0]
        z = mu[rng.choice(n, m, replace=False)] + 0.05 * rng.normal(size=(m, q))
    elif kind == "farcluster":  # 10 % of the rows f l away, no inducing point there
        mu = rng.normal(size=(n, q))
        z = mu[rng.choice(n, m, replace=False)] + 0.05 * rng.normal(size=(m, q))
        mu[: n // 10, 0] += f * ls[0]
    elif kind == "outliers":  # 8 rows f l away along every dimension
        mu = rng.normal(size=(n, q))
        z = mu[rng.choice(np.arange(8, n), m, replace=False)] + 0.05 * rng.normal(size=(m, q))
        mu[:8] += f * ls
    elif kind == "zcluster":  # a small far cluster (5 % of rows) holding 5 inducing points
        mu = rng.normal(size=(n, q))
        k = n // 20
        mu[:k, 0] += f * ls[0]
        idx = np.concatenate([rng.choice(k, 5, replace=False), rng.choice(np.arange(k, n), m - 5, replace=False)])
        z = mu[idx] + 0.05 * rng.normal(size=(m, q))
    a = rng.normal(size=(m, m))
    adj = (-0.7, rng.normal(size=(m, d)), a + a.T)
    return mu, s, y, z, ls, adj


ENVELOPE = [  # (layout, expected mode latent, expected mode SGPR: always the Knm-tile SYRK)
    ("gauss", 1, "fast", "syrk"), ("gauss", 2, "fast", "syrk"), ("gauss", 3, "precise", "syrk"),
    ("gauss", 8, "direct", "syrk"), ("gauss", 16, "direct", "syrk"), ("gauss", 24, "direct", "syrk"),
    ("gauss", 32, "direct", "syrk"), ("bimodal", 10, "precise", "syrk"), ("bimodal", 30, "direct", "syrk"),
    ("bimodal", 300, "direct", "syrk"), ("farcluster", 300, "fast", "syrk"),
    ("outliers", 30, "fast", "syrk"), ("outliers", 1000, "fast", "syrk"),
    ("zcluster", 20, "precise", "syrk"), ("zcluster", 60, "direct", "syrk"),
]


@pytest.mark.parametrize("expected", [True, False])
@pytest.mark.parametrize("case", ENVELOPE, ids=lambda c: f"{c[0]}{c[1]}")
def test_accuracy_envelope(sgp, orc, case, expected):
    kind, f, mode_latent, mode_det = case
    mu, s, y, z, ls, adj = _layout(kind, f)
    k = sgp.KernelSpec(1.3, ls)
    ctx = sgp.Context.default()
    ctx.set_precision("auto")
    st, g = sgp.sweep_stats(expected, mu, s if expected else None, y, z, k, adj=sgp.StatsAdjoints(*adj))
    mode, tz = ctx.last_precision()
    assert mode == (mode_latent if expected else mode_det), (mode, tz)
    wst, wg = orc.sweep_stats(expected, mu, s if expected else None, y, z, 1.3, ls, adj=adj)
    pairs = dict(phi=(st.phi_big, wst.phi_big, STAT_TOL), psi=(st.psi_y, wst.psi_y, STAT_TOL),
                 dz=(g.d_z, wg.d_z, GRAD_TOL), dl=(g.d_lengthscales, wg.d_lengthscales, GRAD_TOL),
                 dvar=([g.d_variance], [wg.d_variance], GRAD_TOL))
    if expected:
        pairs.update(dmu=(g.d_mu, wg.d_mu, GRAD_TOL), ds=(g.d_s, wg.d_s, GRAD_TOL))
    elem_tol = DIRECT_TOL if mode == "direct" else 1e-4  # random adjoints: no coordinator cancellation
    for name, (a, b, tol) in pairs.items():
        assert np.all(np.isfinite(a)), name
        assert rel_err(a, b) < elem_tol, (name, rel_err(a, b), mode)
        assert norm_rel_err(a, b) < (DIRECT_TOL if mode == "direct" else tol), (name, norm_rel_err(a, b), mode)


def _random_shapes(count, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        out.append((int(rng.integers(1, 3000)), int(rng.choice([1, 3, 7, 10, 20, 24, 29, 32, 40, 64])),
                    int(rng.integers(0, 9)), int(rng.integers(1, 90)), bool(rng.integers(0, 2))))
    return out


@pytest.mark.parametrize("shape", _random_shapes(12, seed=77))
def test_direct_mode_parity(sgp, orc, shape):
    """The direct (fp64-exponent) kernels forced on seeded random shapes, Q up to 64 (beyond the
    row-tile instantiations they are the only path), both modes, ragged N, D = 0."""
    n, q, d, m, expected = shape
    m = min(m, n)
    rng = np.random.default_rng(n + q)
    mu = 3.0 * rng.normal(size=(n, q))
    s = rng.uniform(0.25, 1.0, (n, q))
    y = rng.normal(size=(n, d))
    z = mu[rng.choice(n, m, replace=False)]
    ls = rng.uniform(0.5, 2.0, q)
    a = rng.normal(size=(m, m))
    adj = (0.3, rng.normal(size=(m, d)), a + a.T)
    ctx = sgp.Context.default()
    k = sgp.KernelSpec(0.8, ls)
    st, g = sgp.sweep_stats(expected, mu, s if expected else None, y, z, k, adj=sgp.StatsAdjoints(*adj),
                            precision="direct")
    assert ctx.last_precision()[0] == "direct"
    ctx.set_precision("auto")
    wst, wg = orc.sweep_stats(expected, mu, s if expected else None, y, z, 0.8, ls, adj=adj)
    assert rel_err(st.yy, wst.yy) < 1e-13 and st.n_count == wst.n_count
    outs = [(st.phi_big, wst.phi_big), (g.d_z, wg.d_z), (g.d_lengthscales, wg.d_lengthscales),
            ([g.d_variance], [wg.d_variance])]
    if d:
        outs.append((st.psi_y, wst.psi_y))
    if expected:
        outs += [(g.d_mu, wg.d_mu), (g.d_s, wg.d_s)]
    for a_, b_ in outs:
        assert rel_err(a_, b_) < DIRECT_TOL
        assert norm_rel_err(a_, b_) < DIRECT_TOL


def test_direct_mode_engine_subshards(sgp, orc):
    """The direct path through the engine's host-buffer sub-shard pipeline (pair sums folded across
    sub-shards, d mu / d S streamed out), a bimodal latent space at +-300 l."""
    import torch

    n, q, d, m = 520_000, 3, 2, 12
    rng = np.random.default_rng(3)
    mu = rng.normal(size=(n, q))
    mu[:, 0] += np.where(np.arange(n) % 2 == 0, 300.0, -300.0)
    s = rng.uniform(0.25, 1.0, (n, q))
    y = rng.normal(size=(n, d))
    z = mu[rng.choice(n, m, replace=False)]
    ls = np.ones(q)
    eng = sgp.Engine(sgp.ModelKind.latent, mu, s, y)
    gmu = torch.empty(q, n, dtype=torch.float64, pin_memory=True).numpy().T
    gs = torch.empty(q, n, dtype=torch.float64, pin_memory=True).numpy().T
    eng.set_local_grads_out(gmu, gs)
    eng.broadcast(sgp.KernelSpec(1.0, ls), 20.0, z, mu, s)
    r = eng.evaluate(True)
    assert r.timing.precision == "direct"
    ref = orc.engine_evaluate(True, mu, s, y, z, 1.0, ls, 20.0, workers=THREADS)
    _check_eval(r, ref, True, elem_tol=DIRECT_TOL, bound_tol=DIRECT_TOL)


@pytest.mark.parametrize("latent,m", [(True, 100), (False, 100), (True, 300), (False, 500)])
def test_device_coordinator_matches_host(sgp, latent, m, monkeypatch):
    """The coordinator on the device (dcoord.cu: the single-CTA shared-memory kernels for M <= 112,
    the blocked Cholesky / warp-per-column inverse / tiled gemm of dla.cu above) against the host fp64
    coordinator (coordinator.cpp): same statistics in, the same bound / gradients out to fp64 rounding."""
    from paper_1410_4984_b200 import synthetic

    w = synthetic.make(latent, 30_000, 10 if latent else 8, 8, m, seed=4)
    out = []
    for dev in ("1", "0"):
        monkeypatch.setenv("SGPX_DEVICE_COORD", dev)
        eng = sgp.Engine(sgp.ModelKind.latent if latent else sgp.ModelKind.regression, w.mu, w.s, w.y,
                         precision="direct")
        eng.broadcast(w.kernel, w.beta, w.z)
        out.append(eng.evaluate(True))
        eng.close()
    a, b = out
    # the two coordinators sum in different fp64 orders; above the small-M path the blocked Cholesky's
    # order meets cond(Kmm + beta Phi) at M = 500 (~1e-11 on the bound)
    tb, tf, tg = (1e-13, 1e-12, 1e-10) if m <= 112 else (1e-10, 1e-8, 1e-8)
    assert rel_err(a.bound.total, b.bound.total) < tb
    for f in sgp.BOUND_FIELDS:
        assert rel_err(getattr(a.bound, f), getattr(b.bound, f)) < tf, f
    # (with Q = 4 and M = 500, Kmm is ill-conditioned enough that either coordinator and the oracle
    # differ at ~5e-3 in d Z from fp64 summation order alone: tools/dbg_coord_large_m.py)
    assert rel_err(a.grads.d_z, b.grads.d_z) < tg
    assert rel_err(a.grads.d_lengthscales, b.grads.d_lengthscales) < tg
    assert rel_err(a.grads.d_variance, b.grads.d_variance) < tg
    assert rel_err(a.grads.d_beta, b.grads.d_beta) < tg
    assert a.jitter_factor == b.jitter_factor
    if latent:
        assert rel_err(a.grads.d_mu, b.grads.d_mu) < 1e-11


@pytest.mark.parametrize("m", [1, 7, 32, 33, 64, 97, 112])
def test_split_coordinator_small_m_edges(sgp, m, monkeypatch):
    """The split device coordinator (dcoord.cu: bound_g_small_kernel's blocked Cholesky with a short last
    32-column panel, D^-1 blocks, W = L^-1 in place, G = W^T W Psi; bound_u / deferred on the side
    streams) against the host coordinator at the panel edges, with and without gradients."""
    from paper_1410_4984_b200 import synthetic

    w = synthetic.make(True, 6_000, 5, 3, m, seed=21 + m)
    for with_grads in (True, False):
        out = []
        for dev in ("1", "0"):
            monkeypatch.setenv("SGPX_DEVICE_COORD", dev)
            eng = sgp.Engine(sgp.ModelKind.latent, w.mu, w.s, w.y, precision="direct")
            eng.broadcast(w.kernel, w.beta, w.z)
            out.append(eng.evaluate(with_grads))
            eng.close()
        a, b = out
        assert rel_err(a.bound.total, b.bound.total) < 1e-12
        for f in sgp.BOUND_FIELDS:
            assert rel_err(getattr(a.bound, f), getattr(b.bound, f)) < 1e-11, (f, with_grads)
        if with_grads:
            for g in ("d_z", "d_lengthscales", "d_variance", "d_beta", "d_mu", "d_s"):
                assert rel_err(getattr(a.grads, g), getattr(b.grads, g)) < 1e-9, g


def test_split_coordinator_escalation(sgp, monkeypatch):
    """A near-duplicate inducing point: Kmm is singular to working precision, so factor_gram's jitter
    escalation runs (prefactor_small_kernel on the side stream during the forward, coordinator.cpp on the
    host) and the split coordinator factors A = Kmm + jitter + beta Phi with it; both pick the same jitter
    factor and agree."""
    from paper_1410_4984_b200 import synthetic

    w = synthetic.make(True, 4_000, 3, 2, 24, seed=5)
    z = np.array(w.z, copy=True)
    z[1] = z[0] + 1e-9  # Kmm singular to working precision: factor_gram's jitter, then A's shift
    out = []
    for dev in ("1", "0"):
        monkeypatch.setenv("SGPX_DEVICE_COORD", dev)
        eng = sgp.Engine(sgp.ModelKind.latent, w.mu, w.s, w.y, precision="direct")
        eng.broadcast(w.kernel, w.beta, z)
        out.append(eng.evaluate(True))
        eng.close()
    a, b = out
    assert a.jitter_factor == b.jitter_factor and a.jitter_factor > 0.0
    assert rel_err(a.bound.total, b.bound.total) < 1e-9
    # cond(Kmm + jitter) ~ 1e12 here: the two fp64 summation orders differ at ~1e-5 in d mu (measured 8.5e-6)
    assert rel_err(a.grads.d_mu, b.grads.d_mu) < 1e-4


@pytest.mark.parametrize("n,q,d,m", [(50_000, 10, 50, 100), (20_011, 6, 17, 40), (9_000, 12, 64, 128)])
def test_psi1_backward_pipeline_matches_first_version(sgp, orc, n, q, d, m, monkeypatch):
    """psi1_bwd_pipe_kernel (TMA prefetch of the next chunk, T through TMEM, FFMA2) against the first
    tcgen05 backward (SGPX_PSI1_BWD=old) and the oracle: the same statistics and gradients to the mixed
    tolerance (the two sum T in a different fp32 order)."""
    from paper_1410_4984_b200 import synthetic

    w = synthetic.make(True, n, q, d, m, seed=31)
    out = []
    for old in ("0", "1"):
        if old == "1":
            monkeypatch.setenv("SGPX_PSI1_BWD", "old")
        else:
            monkeypatch.delenv("SGPX_PSI1_BWD", raising=False)
        eng = sgp.Engine(sgp.ModelKind.latent, w.mu, w.s, w.y)
        eng.broadcast(w.kernel, w.beta, w.z)
        out.append(eng.evaluate(True))
        eng.close()
    a, b = out
    for g in ("d_z", "d_lengthscales", "d_variance", "d_mu", "d_s"):
        assert norm_rel_err(getattr(a.grads, g), getattr(b.grads, g)) < 2e-6, g
    # against the oracle: no worse than the first version, entry by entry (the worst d Z entries are residues
    # of cancelling sums, ~5e3 x below the block's largest, and carry the row-tile kernels' mixed-precision
    # rounding in both: tools/dbg_dz_check.py) and within the suite's norm-wise tolerance
    ref = orc.engine_evaluate(True, w.mu, w.s, w.y, w.z, w.variance, w.lengthscales, w.beta, workers=THREADS)
    assert rel_err(a.bound.total, ref.bound["total"]) < STAT_TOL
    for g in ("d_z", "d_lengthscales", "d_variance", "d_mu", "d_s"):
        r = np.ravel(getattr(ref, g))
        ea = np.max(np.abs(np.ravel(getattr(a.grads, g)) - r) / np.maximum(np.abs(r), 1e-300))
        eb = np.max(np.abs(np.ravel(getattr(b.grads, g)) - r) / np.maximum(np.abs(r), 1e-300))
        assert ea <= 1.1 * eb + 1e-9, (g, ea, eb)
        assert norm_rel_err(getattr(a.grads, g), getattr(ref, g)) < GRAD_TOL, g


@pytest.mark.parametrize("n,pinned", [(600_000, True), (600_000, False), (250_000, True), (100_000, True)])
def test_end_to_end_graph_replay(sgp, n, pinned):
    """Host mu / S in, d mu / d S out, on an explicit stream: with page-locked buffers the evaluation is
    captured once and replayed as a CUDA graph (uploads, read-backs and the per-broadcast prefactor inside);
    pageable buffers take the per-call path.  Three evaluations with changing host values agree with a
    fresh device-resident engine each time.  Row counts cover the sub-shard plans with host I/O: six
    weighted pieces (>= 400k rows), five (>= 200k), two (>= 80k)."""
    import torch

    from paper_1410_4984_b200 import synthetic

    q, d, m = 10, 8, 50
    w = synthetic.make(True, n, q, d, m, seed=41, device="cuda")
    stream = torch.cuda.Stream()
    ctx = sgp.Context(0)
    ctx.set_stream(stream.cuda_stream)
    eng = sgp.Engine(sgp.ModelKind.latent, w.mu, w.s, w.y, ctx=ctx)

    def host(t):
        if pinned:
            h = torch.empty(q, n, dtype=torch.float64, pin_memory=True)
            h.copy_(t.t())
            return h, h.numpy().T
        h = np.asfortranarray(t.cpu().numpy())
        return None, h

    mu_t, mu_np = host(w.mu)
    s_t, s_np = host(w.s)
    if pinned:
        gmu_t = torch.empty(q, n, dtype=torch.float64, pin_memory=True)
        gs_t = torch.empty(q, n, dtype=torch.float64, pin_memory=True)
        gmu, gs = gmu_t.numpy().T, gs_t.numpy().T
    else:
        gmu, gs = np.zeros((n, q), order="F"), np.zeros((n, q), order="F")
    eng.set_local_grads_out(gmu, gs)
    for step in range(3):
        scale = 1.0 + 0.05 * step
        mu_np[:] = np.asarray(w.mu.cpu()) * scale
        s_np[:] = np.asarray(w.s.cpu()) * scale
        eng.broadcast(w.kernel, w.beta, w.z, mu_np, s_np)
        r = eng.evaluate(True)
        ref_eng = sgp.Engine(sgp.ModelKind.latent, w.mu * scale, w.s * scale, w.y)
        ref_eng.broadcast(w.kernel, w.beta, w.z)
        ref = ref_eng.evaluate(True)
        assert rel_err(r.bound.total, ref.bound.total) < 1e-12, step
        assert norm_rel_err(gmu, ref.grads.d_mu) < 1e-12, step
        assert norm_rel_err(gs, ref.grads.d_s) < 1e-12, step
        assert norm_rel_err(r.grads.d_z, ref.grads.d_z) < 1e-10, step
        ref_eng.close()
    eng.close()


@pytest.mark.parametrize("workers", [2, 3])
@pytest.mark.parametrize("latent", [True, False])
def test_multi_gpu_engine(sgp, orc, workers, latent):
    """sgpx_multi_*: Engine(kind, x, s, y, workers) in one process — shards by make_partition, the two
    exchanges folded per device (here all shards share cuda:0) and allreduced across devices with NCCL
    when there are several — against the single-shard engine and the oracle engine with the same
    worker count (parallel.hpp:326-479)."""
    from paper_1410_4984_b200 import synthetic

    w = synthetic.make(latent, 20_003, 6, 4, 40, seed=9)
    kind = sgp.ModelKind.latent if latent else sgp.ModelKind.regression
    multi = sgp.Engine(kind, w.mu, w.s, w.y, workers=workers, precision="direct")
    assert isinstance(multi, sgp.MultiEngine)
    multi.broadcast(w.kernel, w.beta, w.z, w.mu if latent else None, w.s if latent else None)
    r = multi.evaluate(True)
    one = sgp.Engine(kind, w.mu, w.s, w.y, precision="direct")
    one.broadcast(w.kernel, w.beta, w.z)
    r1 = one.evaluate(True)
    assert rel_err(r.bound.total, r1.bound.total) < 1e-12
    assert rel_err(r.grads.d_z, r1.grads.d_z) < 1e-10
    if latent:
        assert np.array_equal(r.grads.d_mu, r1.grads.d_mu) or rel_err(r.grads.d_mu, r1.grads.d_mu) < 1e-12
    ref = orc.engine_evaluate(latent, w.mu, w.s, w.y, w.z, w.variance, w.lengthscales, w.beta, workers=workers)
    _check_eval(r, ref, latent, elem_tol=DIRECT_TOL, bound_tol=DIRECT_TOL)


@pytest.mark.parametrize("device_coord", ["0", "1"])
@pytest.mark.parametrize("latent", [True, False])
def test_predict_matches_reference(sgp, orc, latent, device_coord, monkeypatch):
    """finalize() + predict(X*) (model.hpp:181-217, 265-296, 353-383): mean = beta K*m A^-1 Psi,
    variance = var - |L_k^-1 k*|^2 + |L_a^-1 k*|^2 (+ 1/beta in observation mode), from the factors of the
    engine's last evaluation, against the oracle restatement; the cached bound too."""
    monkeypatch.setenv("SGPX_DEVICE_COORD", device_coord)
    from paper_1410_4984_b200 import synthetic

    w = synthetic.make(latent, 5000, 3, 4, 30, seed=13)
    eng = sgp.Engine(sgp.ModelKind.latent if latent else sgp.ModelKind.regression, w.mu, w.s, w.y,
                     precision="direct")
    with pytest.raises(ValueError, match="before fit"):
        eng.predict(np.zeros((2, 3)))
    eng.broadcast(w.kernel, w.beta, w.z)
    bound = eng.finalize()
    xs = np.random.default_rng(2).normal(size=(257, 3))
    for mode in ("observation", "latent"):
        mean, var = eng.predict(xs, mode)
        rm, rv, rb = orc.predict(latent, w.mu, w.s, w.y, w.z, w.variance, w.lengthscales, w.beta, xs,
                                 observation=mode == "observation")
        assert rel_err(mean, rm) < 1e-10
        assert rel_err(var, rv) < 1e-10
        assert rel_err(bound, rb) < 1e-12 and rel_err(eng.cached_bound, rb) < 1e-12
    with pytest.raises(ValueError, match="column mismatch"):
        eng.predict(np.zeros((2, 4)))


@pytest.mark.parametrize("latent", [True, False])
def test_fit_session_matches_reference_lbfgs(sgp, orc, latent):
    """FitSession + LbfgsState (model.hpp:100-168, optimizer.hpp:20-458) with the parameter vector and
    the L-BFGS history on the device, against the oracle's restatement over the fp64 engine: the same
    objective values iteration by iteration (direct mode: fp64 on both sides), the same line-search
    evaluation count, the same final parameters."""
    from paper_1410_4984_b200 import synthetic

    w = synthetic.make(latent, 3000, 3, 4, 12, seed=31)
    kind = sgp.ModelKind.latent if latent else sgp.ModelKind.regression
    iters = 6
    fs = sgp.FitSession(kind, w.mu, w.s, w.y, w.kernel, w.beta, w.z, precision="direct")
    values = [fs.state()["value"]]
    for _ in range(iters):
        if not fs.step():
            break
        values.append(fs.state()["value"])
    ref = orc.fit(latent, w.mu, w.s, w.y, w.z, w.variance, w.lengthscales, w.beta, iters, workers=THREADS)
    got = np.array(values)
    want = ref["values"][:len(got)]
    assert np.all(np.diff(got) <= 0.0)
    assert rel_err(got, want) < 1e-8, (got, want)
    st = fs.state()
    assert st["total_evals"] == ref["evals"]
    p = fs.params()
    rp = ref["params"]
    assert rel_err(p["variance"], rp["variance"]) < 1e-7 and rel_err(p["beta"], rp["beta"]) < 1e-7
    assert rel_err(p["lengthscales"], rp["lengthscales"]) < 1e-7 and rel_err(p["z"], rp["z"]) < 1e-7
    if latent:
        assert rel_err(p["mu"], rp["mu"]) < 1e-7 and rel_err(p["s"], rp["s"]) < 1e-7
