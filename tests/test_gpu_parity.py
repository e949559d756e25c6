"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Tolerances (north star: <= 1e-4 relative for the mixed FP32/fp64 path):
  * statistics Phi, Psi, yy:         norm-wise relative error <= 1e-5
  * per-datapoint / global gradients: norm-wise relative error <= 5e-5
  * bound total:                      |a-b| / max(|a|,|b|,1) <= 1e-5 (reference rel_err scale)
The mixed modes (fast / precise) run the exponents as fp16-piece tcgen05 MMAs (psi2) or fp32
direct differences (psi1) with MUFU.EX2; every sum over datapoints and across CTAs is fp64.
"""
import numpy as np
import pytest

from conftest import norm_rel_err, rel_err

pytestmark = pytest.mark.gpu

STAT_TOL = 1e-5
GRAD_TOL = 5e-5
BOUND_TOL = 1e-5


@pytest.fixture(scope="module")
def sgp():
    from paper_1410_4984_b200 import sgp as m

    if m.device_count() == 0:
        pytest.fail("no CUDA device visible to libsgpx (gpu tests must run on the B200)")
    return m


def problem(seed=0, n=300, q=3, d=4, m=7, s_lo=0.25, s_hi=1.0):
    rng = np.random.default_rng(seed)
    mu = rng.normal(size=(n, q))
    s = rng.uniform(s_lo, s_hi, (n, q))
    y = rng.normal(size=(n, d))
    z = mu[rng.choice(n, m, replace=False)] + 0.05 * rng.normal(size=(m, q))
    ls = rng.uniform(0.5, 2.0, q)
    return mu, s, y, z, 1.3, ls


def sym_adj(rng, m, d):
    a = rng.normal(size=(m, m))
    return -0.7, rng.normal(size=(m, d)), a + a.T


@pytest.mark.parametrize("shape", [(300, 3, 4, 7), (1, 1, 1, 1), (33, 2, 1, 5), (257, 10, 10, 100),
                                   (100, 1, 3, 50), (64, 20, 5, 12), (1000, 8, 2, 33), (70, 5, 0, 9)])
@pytest.mark.parametrize("expected", [True, False])
def test_stats_parity(sgp, orc, shape, expected):
    n, q, d, m = shape
    mu, s, y, z, var, ls = problem(1, n, q, d, m)
    k = sgp.KernelSpec(var, ls)
    got = sgp.sweep_stats(expected, mu, s, y, z, k)[0]
    want, _ = orc.sweep_stats(expected, mu, s if expected else None, y, z, var, ls)
    assert got.phi == pytest.approx(want.phi, rel=1e-15)
    assert got.n_count == want.n_count
    assert rel_err(got.yy, want.yy) < 1e-12
    assert norm_rel_err(got.phi_big, want.phi_big) < STAT_TOL
    if d:
        assert norm_rel_err(got.psi_y, want.psi_y) < STAT_TOL
    assert np.array_equal(got.phi_big, got.phi_big.T)


@pytest.mark.parametrize("shape", [(300, 3, 4, 7), (1, 1, 1, 1), (33, 2, 1, 5), (257, 10, 10, 100),
                                   (100, 1, 3, 50), (64, 20, 5, 12), (1000, 8, 2, 33), (64, 12, 5, 12),
                                   (2000, 16, 6, 50), (500, 21, 3, 20), (300, 32, 2, 16)])
@pytest.mark.parametrize("expected", [True, False])
def test_grads_parity(sgp, orc, shape, expected):
    n, q, d, m = shape
    mu, s, y, z, var, ls = problem(2, n, q, d, m)
    rng = np.random.default_rng(5)
    adj = sym_adj(rng, m, d)
    k = sgp.KernelSpec(var, ls)
    st, g = sgp.sweep_stats(expected, mu, s, y, z, k, adj=sgp.StatsAdjoints(*adj))
    wst, wg = orc.sweep_stats(expected, mu, s if expected else None, y, z, var, ls, adj=adj)
    assert norm_rel_err(st.phi_big, wst.phi_big) < STAT_TOL
    assert norm_rel_err(g.d_z, wg.d_z) < GRAD_TOL
    assert rel_err(g.d_variance, wg.d_variance) < GRAD_TOL or norm_rel_err(g.d_variance, wg.d_variance) < GRAD_TOL
    assert norm_rel_err(g.d_lengthscales, wg.d_lengthscales) < GRAD_TOL
    if expected:
        assert norm_rel_err(g.d_mu, wg.d_mu) < GRAD_TOL
        assert norm_rel_err(g.d_s, wg.d_s) < GRAD_TOL


def test_psi1_expected_parity(sgp, orc):
    mu, s, _, z, var, ls = problem(3, 200, 4, 1, 9)
    got = sgp.psi1_expected(sgp.VariationalPosterior(mu, s), z, sgp.KernelSpec(var, ls))
    want = orc.psi1_expected(mu, s, z, var, ls)
    assert rel_err(got, want) < 1e-12


def test_spec_kats_on_gpu(sgp):
    """SPEC.md:130,139,149,158 through the B200 path."""
    k = sgp.KernelSpec(1.0, [1.0])
    st = sgp.stats_deterministic([[0.0]], [[1.0]], [[0.0]], k)
    assert st.phi == 1.0 and abs(st.psi_y[0, 0] - 1.0) < 1e-6 and abs(st.phi_big[0, 0] - 1.0) < 1e-6 and st.yy == 1.0
    q = sgp.VariationalPosterior(np.zeros((1, 1)), np.ones((1, 1)))
    assert abs(sgp.psi1_expected(q, [[0.0]], k)[0, 0] - 1 / np.sqrt(2)) < 1e-15
    assert abs(sgp.psi2_expected(q, [[0.0]], k)[0, 0] - 1 / np.sqrt(3)) < 1e-6
    assert sgp.psi0_expected(sgp.VariationalPosterior(np.zeros((10, 1)), np.ones((10, 1))), sgp.KernelSpec(2.0, [1.0])) == 20.0


def test_errors_match_reference(sgp):
    k = sgp.KernelSpec(1.0, [1.0])
    with pytest.raises(ValueError, match="variances must be positive"):
        sgp.stats_expected(sgp.VariationalPosterior(np.zeros((4, 1)), np.zeros((4, 1))), np.zeros((4, 1)), [[0.0]], k)
    bad = np.zeros((4, 1))
    bad[2, 0] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        sgp.stats_deterministic(bad, np.zeros((4, 1)), [[0.0]], k)
    with pytest.raises(ValueError, match="symmetric"):
        sgp.sweep_stats(True, np.zeros((4, 1)), np.ones((4, 1)), np.zeros((4, 1)), [[0.0], [1.0]], k,
                        adj=sgp.StatsAdjoints(0.0, np.zeros((2, 1)), np.array([[0.0, 1.0], [0.0, 0.0]])))
    with pytest.raises(ValueError, match="kernel dimension"):
        sgp.stats_deterministic(np.zeros((4, 2)), np.zeros((4, 1)), np.zeros((1, 2)), k)
    # N == 0: zero statistics, no launch
    st = sgp.stats_deterministic(np.zeros((0, 1)), np.zeros((0, 2)), [[0.0]], k)
    assert st.phi == 0.0 and st.n_count == 0 and np.all(st.phi_big == 0)


def test_bitwise_determinism(sgp):
    mu, s, y, z, var, ls = problem(4, 5000, 10, 10, 100)
    k = sgp.KernelSpec(var, ls)
    rng = np.random.default_rng(0)
    adj = sgp.StatsAdjoints(*sym_adj(rng, 100, 10))
    a = sgp.sweep_stats(True, mu, s, y, z, k, adj=adj)
    b = sgp.sweep_stats(True, mu, s, y, z, k, adj=adj)
    assert np.array_equal(a[0].phi_big, b[0].phi_big) and np.array_equal(a[0].psi_y, b[0].psi_y)
    assert np.array_equal(a[1].d_mu, b[1].d_mu) and np.array_equal(a[1].d_z, b[1].d_z)


@pytest.mark.parametrize("latent", [True, False])
@pytest.mark.parametrize("shape", [(3000, 10, 10, 100), (2500, 7, 4, 60), (1500, 13, 3, 140)])
def test_engine_evaluate_parity(sgp, orc, latent, shape):
    """Engine::evaluate(true): bound and every gradient segment vs the oracle engine (exact and
    padded Q, psi1 on the tile and on the M > 128 kernels)."""
    n, q, d, m = shape
    mu, s, y, z, var, ls = problem(6, n, q, d, m)
    beta = 100.0
    k = sgp.KernelSpec(var, ls)
    eng = sgp.Engine(sgp.ModelKind.latent if latent else sgp.ModelKind.regression, mu, s if latent else None, y)
    eng.broadcast(k, beta, z)
    r = eng.evaluate(True)
    ref = orc.engine_evaluate(latent, mu, s, y, z, var, ls, beta, workers=4)
    assert rel_err(r.bound.total, ref.bound["total"]) < BOUND_TOL
    for f in sgp.BOUND_FIELDS:
        assert rel_err(getattr(r.bound, f), ref.bound[f]) < BOUND_TOL, f
    g = r.grads
    assert norm_rel_err(g.d_z, ref.d_z) < GRAD_TOL
    assert norm_rel_err(g.d_lengthscales, ref.d_lengthscales) < GRAD_TOL
    assert rel_err(g.d_variance, ref.d_variance) < GRAD_TOL * max(1.0, abs(ref.d_variance)) ** 0 or \
        norm_rel_err(g.d_variance, ref.d_variance) < GRAD_TOL
    assert norm_rel_err(g.d_beta, ref.d_beta) < GRAD_TOL
    if latent:
        assert norm_rel_err(g.d_mu, ref.d_mu) < GRAD_TOL
        assert norm_rel_err(g.d_s, ref.d_s) < GRAD_TOL


@pytest.mark.parametrize("shape", [(100000, 8, 50, 48), (30000, 10, 50, 100), (2000, 20, 6, 256), (20000, 18, 10, 64)])
def test_multi_chunk_parity(sgp, orc, shape):
    """Shards large enough that every CTA of every kernel walks many chunks (pipelined producer /
    consumer rings wrap several times; psi1 tiles exceed one per thread)."""
    n, q, d, m = shape
    mu, s, y, z, var, ls = problem(7, n, q, d, m)
    rng = np.random.default_rng(8)
    adj = sym_adj(rng, m, d)
    k = sgp.KernelSpec(var, ls)
    st, g = sgp.sweep_stats(True, mu, s, y, z, k, adj=sgp.StatsAdjoints(*adj))
    wst, wg = orc.sweep_stats(True, mu, s, y, z, var, ls, adj=adj)
    assert rel_err(st.yy, wst.yy) < 1e-12
    assert norm_rel_err(st.phi_big, wst.phi_big) < STAT_TOL
    assert norm_rel_err(st.psi_y, wst.psi_y) < STAT_TOL
    assert norm_rel_err(g.d_z, wg.d_z) < GRAD_TOL
    assert norm_rel_err(g.d_lengthscales, wg.d_lengthscales) < GRAD_TOL
    assert rel_err(g.d_variance, wg.d_variance) < GRAD_TOL
    assert norm_rel_err(g.d_mu, wg.d_mu) < GRAD_TOL
    assert norm_rel_err(g.d_s, wg.d_s) < GRAD_TOL


def _random_shapes(count=10, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        out.append((int(rng.integers(1, 5000)), int(rng.choice([1, 2, 3, 5, 7, 9, 10, 11, 13, 16, 17, 20])),
                    int(rng.integers(0, 13)), int(rng.integers(1, 141)), bool(rng.integers(0, 2))))
    return out


@pytest.mark.parametrize("shape", _random_shapes(8, seed=99))
def test_random_engine_parity(sgp, orc, shape):
    """Engine::evaluate(true) on seeded random shapes / modes: bound, KL, d beta and every gradient."""
    n, q, d, m, latent = shape
    d = max(d, 1)
    m = min(m, n)
    mu, s, y, z, var, ls = problem(41, n, q, d, m)
    k = sgp.KernelSpec(var, ls)
    eng = sgp.Engine(sgp.ModelKind.latent if latent else sgp.ModelKind.regression, mu, s if latent else None, y)
    eng.broadcast(k, 30.0, z)
    r = eng.evaluate(True)
    ref = orc.engine_evaluate(latent, mu, s, y, z, var, ls, 30.0, workers=4)
    assert rel_err(r.bound.total, ref.bound["total"]) < BOUND_TOL
    g = r.grads
    assert norm_rel_err(g.d_z, ref.d_z) < GRAD_TOL
    assert norm_rel_err(g.d_lengthscales, ref.d_lengthscales) < GRAD_TOL
    assert rel_err(g.d_variance, ref.d_variance) < GRAD_TOL or norm_rel_err(g.d_variance, ref.d_variance) < GRAD_TOL
    assert norm_rel_err(g.d_beta, ref.d_beta) < GRAD_TOL
    if latent:
        assert norm_rel_err(g.d_mu, ref.d_mu) < GRAD_TOL
        assert norm_rel_err(g.d_s, ref.d_s) < GRAD_TOL


@pytest.mark.parametrize("shape", _random_shapes(6, seed=5))
def test_random_shapes_precise_mode(sgp, orc, shape):
    """Wide latent spread (mu ~ N(0, 4^2): spread^2 >> 60) selects the precise mode (three-piece
    MMA1, fp16 forward MMA3) on random shapes, padded Q included; expected mode."""
    n, q, d, m, _ = shape
    m = min(m, n)
    mu, s, y, z, var, ls = problem(51, n, q, d, m)
    mu, z = 4.0 * mu, 4.0 * z
    adj = sym_adj(np.random.default_rng(52), m, d)
    k = sgp.KernelSpec(var, ls)
    st, g = sgp.sweep_stats(True, mu, s, y, z, k, adj=sgp.StatsAdjoints(*adj))
    wst, wg = orc.sweep_stats(True, mu, s, y, z, var, ls, adj=adj)
    assert norm_rel_err(st.phi_big, wst.phi_big) < 3e-5
    if d > 0:
        assert norm_rel_err(st.psi_y, wst.psi_y) < STAT_TOL
    assert norm_rel_err(g.d_z, wg.d_z) < GRAD_TOL
    assert norm_rel_err(g.d_lengthscales, wg.d_lengthscales) < GRAD_TOL
    assert rel_err(g.d_variance, wg.d_variance) < GRAD_TOL or norm_rel_err(g.d_variance, wg.d_variance) < GRAD_TOL
    assert norm_rel_err(g.d_mu, wg.d_mu) < GRAD_TOL
    assert norm_rel_err(g.d_s, wg.d_s) < GRAD_TOL


@pytest.mark.parametrize("shape", _random_shapes() + _random_shapes(12, seed=7))
def test_random_shapes_parity(sgp, orc, shape):
    """Seeded random (N, Q, D, M, mode): ragged N (not a multiple of any chunk), Q between the
    instantiated widths, D = 0 allowed, M up to 140 (psi1 beyond the 128-wide tile)."""
    n, q, d, m, expected = shape
    m = min(m, n)  # Z = distinct rows of mu
    mu, s, y, z, var, ls = problem(31, n, q, d, m)
    adj = sym_adj(np.random.default_rng(32), m, d)
    k = sgp.KernelSpec(var, ls)
    st, g = sgp.sweep_stats(expected, mu, s if expected else None, y, z, k, adj=sgp.StatsAdjoints(*adj))
    wst, wg = orc.sweep_stats(expected, mu, s if expected else None, y, z, var, ls, adj=adj)
    assert norm_rel_err(st.phi_big, wst.phi_big) < STAT_TOL
    if d > 0:
        assert norm_rel_err(st.psi_y, wst.psi_y) < STAT_TOL
    assert norm_rel_err(g.d_z, wg.d_z) < GRAD_TOL
    assert norm_rel_err(g.d_lengthscales, wg.d_lengthscales) < GRAD_TOL
    assert rel_err(g.d_variance, wg.d_variance) < GRAD_TOL or norm_rel_err(g.d_variance, wg.d_variance) < GRAD_TOL
    if expected:
        assert norm_rel_err(g.d_mu, wg.d_mu) < GRAD_TOL
        assert norm_rel_err(g.d_s, wg.d_s) < GRAD_TOL


@pytest.mark.parametrize("shape", [(100000, 8, 1, 48), (3000, 8, 1, 500), (20000, 12, 3, 100),
                                   (20000, 16, 2, 64)])
def test_sgpr_multi_chunk_parity(sgp, orc, shape):
    """Deterministic (SGPR) mode on the row-tile path (precise mode, Q <= 16), many chunks per CTA;
    (3000, 8, 1, 500) is the C4 shape at an oracle-sized N (125,250 pairs)."""
    n, q, d, m = shape
    x, _, y, z, var, ls = problem(11, n, q, d, m)
    rng = np.random.default_rng(12)
    adj = sym_adj(rng, m, d)
    k = sgp.KernelSpec(var, ls)
    st, g = sgp.sweep_stats(False, x, None, y, z, k, adj=sgp.StatsAdjoints(*adj))
    wst, wg = orc.sweep_stats(False, x, None, y, z, var, ls, adj=adj)
    assert norm_rel_err(st.phi_big, wst.phi_big) < STAT_TOL
    assert norm_rel_err(st.psi_y, wst.psi_y) < STAT_TOL
    assert norm_rel_err(g.d_z, wg.d_z) < GRAD_TOL
    assert norm_rel_err(g.d_lengthscales, wg.d_lengthscales) < GRAD_TOL
    assert rel_err(g.d_variance, wg.d_variance) < GRAD_TOL


@pytest.mark.parametrize("spread", [1.0, 2.0, 8.0, 16.0])
def test_data_spread_envelope(sgp, orc, spread):
    """mu ~ N(0, spread^2) with Z drawn from mu and l in [0.5, 2]: the exponent-as-GEMM features
    grow like (mu / l)^2 and cancel for nearby pairs, so the 2^-22 piece accuracy becomes an
    absolute exponent error ~ 2^-22 Q (spread / l)^2.  Within spread 2 l the fast
    mode (two-piece MMA1, bf16 forward MMA3) holds the default tolerances; beyond it the spread check
    selects the precise mode (three-piece MMA1, scaled fp16 forward MMA3), which keeps the gradients
    within GRAD_TOL at spread 8 (measured dz 1.1e-5, Phi 1.5e-5) and within the north star's 1e-4
    at spread 16 (dz 3.5e-5, dS 4.1e-5, Phi 7.3e-5; profiles/accuracy/r01_spread_precise.log)."""
    n, q, d, m = 4000, 10, 10, 100
    rng = np.random.default_rng(1)
    mu = spread * rng.normal(size=(n, q))
    s = rng.uniform(0.25, 1.0, (n, q))
    y = rng.normal(size=(n, d))
    z = mu[rng.choice(n, m, replace=False)] + 0.05 * rng.normal(size=(m, q))
    ls = rng.uniform(0.5, 2.0, q)
    adj = sym_adj(rng, m, d)
    k = sgp.KernelSpec(1.3, ls)
    st, g = sgp.sweep_stats(True, mu, s, y, z, k, adj=sgp.StatsAdjoints(*adj))
    wst, wg = orc.sweep_stats(True, mu, s, y, z, 1.3, ls, adj=adj)
    stat_tol, grad_tol = {1.0: (STAT_TOL, GRAD_TOL), 2.0: (STAT_TOL, GRAD_TOL), 8.0: (3e-5, GRAD_TOL),
                          16.0: (1e-4, 1e-4)}[spread]
    assert norm_rel_err(st.phi_big, wst.phi_big) < stat_tol
    assert norm_rel_err(st.psi_y, wst.psi_y) < stat_tol
    assert norm_rel_err(g.d_mu, wg.d_mu) < grad_tol
    assert norm_rel_err(g.d_s, wg.d_s) < grad_tol
    assert norm_rel_err(g.d_lengthscales, wg.d_lengthscales) < grad_tol
    assert norm_rel_err(g.d_z, wg.d_z) < grad_tol


@pytest.mark.parametrize("q", [4, 7])
@pytest.mark.parametrize("spread", [1.0, 8.0])
def test_engine_subshard_pipeline(sgp, spread, q):
    """Host-resident mu / S (streamed per sub-shard with the kernels) and registered host
    gradient outputs give the same evaluation as the device-resident single pass.  spread 8
    selects the precise mode (host-sample decision for the streamed path, device reduction for the
    resident one); its forward Y scales are per sub-shard, so the two runs agree to the fp16-piece
    rounding instead of bitwise."""
    import torch

    n, d, m = 600_000, 3, 24  # >= 400k rows: six weighted sub-shards with host I/O
    mu, s, y, z, var, ls = problem(9, n, q, d, m)
    mu = mu * spread
    z = z * spread
    k = sgp.KernelSpec(var, ls)
    dev = torch.device("cuda", 0)
    ctx = sgp.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    # device-resident reference run
    mu_t = torch.from_numpy(np.asfortranarray(mu)).to(dev).t().contiguous().t()
    s_t = torch.from_numpy(np.asfortranarray(s)).to(dev).t().contiguous().t()
    y_t = torch.from_numpy(np.asfortranarray(y)).to(dev).t().contiguous().t()
    e1 = sgp.Engine(sgp.ModelKind.latent, mu_t, s_t, y_t, ctx=ctx)
    e1.broadcast(k, 50.0, z, mu_t, s_t)
    r1 = e1.evaluate(True)
    # host path: deferred, streamed upload + registered (pinned) gradient outputs
    e2 = sgp.Engine(sgp.ModelKind.latent, mu, s, y, ctx=ctx)
    gmu = torch.empty(q, n, dtype=torch.float64, pin_memory=True).numpy().T
    gs = torch.empty(q, n, dtype=torch.float64, pin_memory=True).numpy().T
    e2.set_local_grads_out(gmu, gs)
    for _ in range(2):  # second evaluation reuses the registered buffers
        e2.broadcast(k, 50.0, z, mu, s)
        r2 = e2.evaluate(True)
    tb, tg, tl = (1e-12, 1e-10, 1e-13) if spread == 1.0 else (1e-7, 2e-5, 1e-6)
    assert rel_err(r2.bound.total, r1.bound.total) < tb
    assert norm_rel_err(r2.grads.d_z, r1.grads.d_z) < tg
    assert norm_rel_err(r2.grads.d_lengthscales, r1.grads.d_lengthscales) < tg
    assert r2.grads.d_mu is gmu and r2.grads.d_s is gs
    assert norm_rel_err(gmu, r1.grads.d_mu) < tl and norm_rel_err(gs, r1.grads.d_s) < tl


@pytest.mark.parametrize("shape", [(5000, 10, 64, 128), (3001, 6, 65, 100), (2000, 4, 128, 40), (2000, 4, 129, 40),
                                   (3, 2, 3, 2), (4097, 3, 17, 129)])
@pytest.mark.parametrize("precision", ["fast", "precise"])
def test_psi1_tensor_core_limits(sgp, orc, shape, precision, monkeypatch):
    """The tcgen05 psi1 kernels at and past their limits (M <= 128; D <= 128 forward, D <= 64 backward;
    past them the SIMT tile / row kernels take over) against the oracle, and the tensor-core path
    against the SIMT tile kernels (SGPX_PSI1=simt) on the same inputs."""
    n, q, d, m = shape
    mu, s, y, z, var, ls = problem(17, n, q, d, m)
    rng = np.random.default_rng(18)
    adj = sym_adj(rng, m, d)
    k = sgp.KernelSpec(var, ls)
    st, g = sgp.sweep_stats(True, mu, s, y, z, k, adj=sgp.StatsAdjoints(*adj), precision=precision)
    wst, wg = orc.sweep_stats(True, mu, s, y, z, var, ls, adj=adj)
    assert rel_err(st.yy, wst.yy) < 1e-12
    assert norm_rel_err(st.psi_y, wst.psi_y) < STAT_TOL
    assert norm_rel_err(st.phi_big, wst.phi_big) < STAT_TOL
    for a, b in ((g.d_z, wg.d_z), (g.d_lengthscales, wg.d_lengthscales), (g.d_mu, wg.d_mu), (g.d_s, wg.d_s)):
        assert norm_rel_err(a, b) < GRAD_TOL
    monkeypatch.setenv("SGPX_PSI1", "simt")
    st2, g2 = sgp.sweep_stats(True, mu, s, y, z, k, adj=sgp.StatsAdjoints(*adj), precision=precision)
    assert norm_rel_err(st.psi_y, st2.psi_y) < STAT_TOL
    assert norm_rel_err(g.d_mu, g2.d_mu) < GRAD_TOL and norm_rel_err(g.d_z, g2.d_z) < GRAD_TOL
