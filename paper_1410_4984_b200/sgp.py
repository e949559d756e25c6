"""Reference-facing API of the B200 psi-statistics engine.

Mirrors the public surface of the reference's hot path (same names, argument
meaning and error behaviour) over the C ABI of ``include/sgpx.h``:

  reference (proj/include/sgp/...)                 here
  ----------------------------------------------   -------------------------------
  KernelSpec               kernels.hpp:13-33       KernelSpec
  TileConfig               common.hpp:30-37        TileConfig
  VariationalPosterior     psi_stats.hpp:13-26     VariationalPosterior
  SufficientStats          psi_stats.hpp:31-53     SufficientStats
  StatsAdjoints            psi_stats.hpp:56-60     StatsAdjoints
  StatsGrads               psi_stats.hpp:65-71     StatsGrads
  detail::sweep_stats      psi_stats.hpp:108-326   sweep_stats
  stats_deterministic      psi_stats.hpp:332-340   stats_deterministic
  psi0/1/2_expected        psi_stats.hpp:343-386   psi0_expected / psi1_expected / psi2_expected
  stats_expected           psi_stats.hpp:389-397   stats_expected
  stats_grads(+_determ.)   psi_stats.hpp:402-426   stats_grads / stats_grads_deterministic
  make_partition           parallel.hpp:28-41      make_partition
  Engine                   parallel.hpp:326-479    Engine (one GPU; ranks: engine_dist.DistributedEngine)
  BoundBreakdown           bound.hpp:22-35         BoundBreakdown

Errors: std::invalid_argument -> SgpxInvalidArgument (a ValueError),
sgp::NumericError -> SgpxNumericError.  Matrices are numpy float64 (any
layout; copied to column-major) or CUDA torch tensors with unit row stride.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _lib as L
from ._lib import SgpxCudaError, SgpxError, SgpxInvalidArgument, SgpxNumericError, check  # noqa: F401

# ---------------------------------------------------------------------------
# value types
# ---------------------------------------------------------------------------


@dataclass
class KernelSpec:
    """ARD exponentiated quadratic: variance * exp(-1/2 sum_q (x_q - x'_q)^2 / l_q^2)."""
    variance: float = 1.0
    lengthscales: np.ndarray = field(default_factory=lambda: np.ones(1))

    def __post_init__(self):
        self.lengthscales = np.ascontiguousarray(np.atleast_1d(np.asarray(self.lengthscales, dtype=np.float64)))

    def input_dim(self) -> int:
        return int(self.lengthscales.size)

    @staticmethod
    def iso(variance: float, lengthscale: float, q: int) -> "KernelSpec":
        return KernelSpec(variance, np.full(q, float(lengthscale)))

    def _c(self):
        ks = L.kernel_spec(float(self.variance), self.lengthscales.ctypes.data_as(C.c_void_p), self.input_dim())
        return ks


@dataclass
class TileConfig:
    """Accepted for API parity; validated (>= 1) and otherwise ignored — the sm_100a
    launch geometry replaces the reference's CPU block/thread emulation."""
    block_span: int = 64
    thread_span: int = 1024

    def _c(self):
        return L.tile_config(int(self.block_span), int(self.thread_span))


@dataclass
class VariationalPosterior:
    mu: np.ndarray
    s: np.ndarray

    def n(self):
        return self.mu.shape[0]

    def q(self):
        return self.mu.shape[1]


@dataclass
class SufficientStats:
    phi: float = 0.0
    psi_y: np.ndarray | None = None
    phi_big: np.ndarray | None = None
    yy: float = 0.0
    n_count: int = 0

    def __iadd__(self, o: "SufficientStats"):
        self.phi += o.phi
        self.psi_y = self.psi_y + o.psi_y
        self.phi_big = self.phi_big + o.phi_big
        self.yy += o.yy
        self.n_count += o.n_count
        return self


@dataclass
class StatsAdjoints:
    d_phi: float
    d_psi_y: np.ndarray
    d_phi_big: np.ndarray


@dataclass
class StatsGrads:
    d_mu: np.ndarray | None = None
    d_s: np.ndarray | None = None
    d_z: np.ndarray | None = None
    d_variance: float = 0.0
    d_lengthscales: np.ndarray | None = None


BOUND_FIELDS = ("total", "log_det_term", "data_fit_term", "quadratic_term", "trace_phi_term", "trace_kmm_term",
                "kl_term")


@dataclass
class BoundBreakdown:
    total: float = 0.0
    log_det_term: float = 0.0
    data_fit_term: float = 0.0
    quadratic_term: float = 0.0
    trace_phi_term: float = 0.0
    trace_kmm_term: float = 0.0
    kl_term: float = 0.0

    def term_sum(self):
        return (self.log_det_term + self.data_fit_term + self.quadratic_term + self.trace_phi_term +
                self.trace_kmm_term + self.kl_term)

    @staticmethod
    def _from(b: L.bound_breakdown) -> "BoundBreakdown":
        return BoundBreakdown(*(getattr(b, f) for f in BOUND_FIELDS))


class ModelKind(IntEnum):
    regression = 0
    latent = 1


# ---------------------------------------------------------------------------
# matrices at the boundary
# ---------------------------------------------------------------------------
def _F(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _cm(a: np.ndarray) -> L.cmat:
    a2 = a if a.ndim == 2 else a.reshape(a.shape[0], -1)
    return L.cmat(a2.ctypes.data_as(C.c_void_p) if a2.size else None, a2.shape[0], a2.shape[1], a2.shape[0])


_EMPTY = np.zeros((0, 0), order="F")


def _is_cuda_tensor(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def device_view(t) -> L.cmat:
    """Column-major view of a CUDA float64 torch tensor of shape (rows, cols) with stride (1, ld)."""
    import torch

    if t.dtype != torch.float64:
        raise SgpxInvalidArgument("device matrices must be float64")
    rows, cols = t.shape
    if rows > 1 and cols > 1 and t.stride(0) != 1:
        raise SgpxInvalidArgument("device matrices must be column-major (stride(0) == 1); use device_matrix()")
    ld = t.stride(1) if cols > 1 else rows
    return L.cmat(t.data_ptr(), rows, cols, max(ld, rows))


def device_matrix(a, device="cuda"):
    """Copy a host matrix to a column-major float64 CUDA tensor (shape rows x cols)."""
    import torch

    a = np.asarray(a, dtype=np.float64)
    return torch.from_numpy(np.ascontiguousarray(a.T)).to(device).t()


# ---------------------------------------------------------------------------
# contexts
# ---------------------------------------------------------------------------
class Context:
    """One device + one stream + scratch (sgpx_ctx).  Single-threaded."""

    _tls = threading.local()

    def __init__(self, device: int = 0):
        lib = L.load()
        h = C.c_void_p()
        check(lib.sgpx_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = device
        self._lib = lib

    def set_stream(self, stream_ptr: int):
        check(self._lib.sgpx_ctx_set_stream(self.handle, C.c_void_p(stream_ptr)))

    def synchronize(self):
        check(self._lib.sgpx_ctx_synchronize(self.handle))

    def launch_count(self) -> int:
        return int(self._lib.sgpx_ctx_launch_count(self.handle))

    def set_precision(self, precision: str | int = "auto"):
        """Precision mode of the one-shot entry points: "auto" | "fast" | "precise" | "direct"."""
        check(self._lib.sgpx_ctx_set_precision(self.handle, precision_code(precision)))

    def last_precision(self):
        """(mode name, Tz) of the last sweep_stats on this context."""
        tz = C.c_double()
        mode = int(self._lib.sgpx_ctx_last_precision(self.handle, C.byref(tz)))
        return L.PRECISION_NAMES.get(mode, "none"), tz.value

    def close(self):
        if getattr(self, "handle", None):
            self._lib.sgpx_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        d = getattr(cls._tls, "ctxs", None)
        if d is None:
            d = cls._tls.ctxs = {}
        if device not in d:
            d[device] = Context(device)
        return d[device]


def precision_code(precision) -> int:
    if isinstance(precision, str):
        codes = {v: k for k, v in L.PRECISION_NAMES.items()}
        if precision not in codes:
            raise SgpxInvalidArgument(f"unknown precision mode {precision!r}")
        return codes[precision]
    return int(precision)


def device_count() -> int:
    return int(L.load().sgpx_device_count())


# ---------------------------------------------------------------------------
# the sweep and its wrappers (psi_stats.hpp:108-426)
# ---------------------------------------------------------------------------
def sweep_stats(expected: bool, mu, s, y, z, kernel: KernelSpec, tiles: TileConfig | None = None,
                adj: StatsAdjoints | None = None, want_grads: bool = False, ctx: Context | None = None,
                precision: str | None = None):
    """detail::sweep_stats on the B200: returns (SufficientStats, StatsGrads | None).
    ``precision`` (optional) sets the context's mode for this and later calls."""
    ctx = ctx or Context.default()
    if precision is not None:
        ctx.set_precision(precision)
    mu = _F(mu)
    y = _F(y)
    z = _F(z)
    n, q = mu.shape
    m = z.shape[0]
    d = y.shape[1]
    s = _F(s) if expected else _EMPTY
    st = SufficientStats(psi_y=np.zeros((m, d), order="F"), phi_big=np.zeros((m, m), order="F"))
    cst = L.sufficient_stats(0.0, _cm(st.psi_y), _cm(st.phi_big), 0.0, 0)
    cadj = None
    if adj is not None:
        dpsi, dphi = _F(adj.d_psi_y), _F(adj.d_phi_big)
        cadj = L.stats_adjoints(float(adj.d_phi), _cm(dpsi), _cm(dphi))
    g = None
    cg = None
    if want_grads or adj is not None:
        g = StatsGrads(d_mu=np.zeros((n, q), order="F") if expected else None,
                       d_s=np.zeros((n, q), order="F") if expected else None,
                       d_z=np.zeros((m, q), order="F"), d_lengthscales=np.zeros(q))
        cg = L.stats_grads(_cm(g.d_mu) if expected else L.cmat(None, 0, 0, 0),
                           _cm(g.d_s) if expected else L.cmat(None, 0, 0, 0), _cm(g.d_z), 0.0,
                           g.d_lengthscales.ctypes.data_as(C.c_void_p))
    tiles = tiles or TileConfig()
    ks = kernel._c()
    tc = tiles._c()
    check(L.load().sgpx_sweep_stats(ctx.handle, 1 if expected else 0, _cm(mu), _cm(s), _cm(y), _cm(z), C.byref(ks),
                                    C.byref(tc), C.byref(cadj) if cadj is not None else None, C.byref(cst),
                                    C.byref(cg) if cg is not None else None))
    st.phi, st.yy, st.n_count = cst.phi, cst.yy, int(cst.n_count)
    if g is not None:
        g.d_variance = cg.d_variance
    return st, g


def stats_deterministic(x, y, z, kernel: KernelSpec, tiles: TileConfig | None = None, ctx=None) -> SufficientStats:
    return sweep_stats(False, x, None, y, z, kernel, tiles, ctx=ctx)[0]


def psi0_expected(q: VariationalPosterior, kernel: KernelSpec) -> float:
    out = C.c_double()
    mu, s = _F(q.mu), _F(q.s)
    ks = kernel._c()
    check(L.load().sgpx_psi0_expected(_cm(mu), _cm(s), C.byref(ks), C.byref(out)))
    return out.value


def psi1_expected(q: VariationalPosterior, z, kernel: KernelSpec, ctx=None) -> np.ndarray:
    ctx = ctx or Context.default()
    mu, s, z = _F(q.mu), _F(q.s), _F(z)
    out = np.zeros((mu.shape[0], z.shape[0]), order="F")
    ks = kernel._c()
    check(L.load().sgpx_psi1_expected(ctx.handle, _cm(mu), _cm(s), _cm(z), C.byref(ks), _cm(out)))
    return out


def psi2_expected(q: VariationalPosterior, z, kernel: KernelSpec, tiles: TileConfig | None = None,
                  ctx=None) -> np.ndarray:
    y = np.zeros((q.mu.shape[0], 0), order="F")
    return sweep_stats(True, q.mu, q.s, y, z, kernel, tiles, ctx=ctx)[0].phi_big


def stats_expected(q: VariationalPosterior, y, z, kernel: KernelSpec, tiles: TileConfig | None = None,
                   ctx=None) -> SufficientStats:
    return sweep_stats(True, q.mu, q.s, y, z, kernel, tiles, ctx=ctx)[0]


def stats_grads(q: VariationalPosterior, y, z, kernel: KernelSpec, adj: StatsAdjoints,
                tiles: TileConfig | None = None, stats_out: list | None = None, ctx=None) -> StatsGrads:
    st, g = sweep_stats(True, q.mu, q.s, y, z, kernel, tiles, adj=adj, ctx=ctx)
    if stats_out is not None:
        stats_out.append(st)
    return g


def stats_grads_deterministic(x, y, z, kernel: KernelSpec, adj: StatsAdjoints, tiles: TileConfig | None = None,
                              stats_out: list | None = None, ctx=None) -> StatsGrads:
    st, g = sweep_stats(False, x, None, y, z, kernel, tiles, adj=adj, ctx=ctx)
    if stats_out is not None:
        stats_out.append(st)
    return g


# ---------------------------------------------------------------------------
# partition + engine (parallel.hpp)
# ---------------------------------------------------------------------------
def make_partition(n: int, p: int):
    """Balanced contiguous shards, remainder to the earliest (parallel.hpp:28-41)."""
    if p < 1:
        raise SgpxInvalidArgument("make_partition: worker count must be >= 1")
    if p > n:
        raise SgpxInvalidArgument("make_partition: more workers than datapoints")
    base, rem = divmod(n, p)
    out, at = [], 0
    for i in range(p):
        ln = base + (1 if i < rem else 0)
        out.append((at, at + ln))
        at += ln
    return out


@dataclass
class GradientParts:
    d_mu: object = None
    d_s: object = None
    d_z: np.ndarray | None = None
    d_variance: float = 0.0
    d_lengthscales: np.ndarray | None = None
    d_beta: float = 0.0


@dataclass
class EngineTimings:
    stats_pass_s: float = 0.0
    coordinator_s: float = 0.0
    grad_pass_s: float = 0.0
    wall_s: float = 0.0
    fwd_kernel_s: float = 0.0
    bwd_kernel_s: float = 0.0
    fwd_grid: int = 0
    bwd_grid: int = 0
    precision: str = "auto"
    z_spread: float = 0.0
    psi2_fwd_kernel_s: float = 0.0
    psi2_bwd_kernel_s: float = 0.0


@dataclass
class EvalResult:
    bound: BoundBreakdown
    stats: SufficientStats
    has_grads: bool
    grads: GradientParts
    timing: EngineTimings
    jitter_factor: float = 0.0


class Engine:
    """sgp::Engine on one B200 (parallel.hpp:326-479).

    ``Engine(kind, x_or_mu, s, y, workers=1, tiles=TileConfig(), jitter_factor=1e-6)``.
    Rows stay resident in HBM; ``broadcast`` sets (kernel, beta, Z) and optionally new
    (mu, s); ``evaluate(with_grads)`` runs forward kernel -> fp64 coordinator ->
    backward kernel.  ``workers`` > 1 is served by ``engine_dist.DistributedEngine``
    (one rank per GPU, NCCL allreduce); on a single device it must be 1.
    """

    def __new__(cls, kind, x_or_mu, s, y, workers: int = 1, *args, **kwargs):
        if cls is Engine and workers != 1:
            return MultiEngine(kind, x_or_mu, s, y, workers, *args, **kwargs)
        return super().__new__(cls)

    def __init__(self, kind, x_or_mu, s, y, workers: int = 1, tiles: TileConfig | None = None,
                 jitter_factor: float = 1e-6, ctx: Context | None = None, _n_global=None, _row_begin=0,
                 precision: str = "auto"):
        self.kind = ModelKind(kind)
        if workers != 1:
            raise SgpxInvalidArgument("Engine(workers > 1) is the multi-GPU engine (MultiEngine)")
        (tiles or TileConfig())  # accepted, geometry is fixed
        self.ctx = ctx or Context.default()
        self._lib = L.load()
        on_dev = _is_cuda_tensor(y)
        n, d = y.shape
        q = x_or_mu.shape[1]
        self.n, self.d, self.q = n, d, q
        self.n_global = n if _n_global is None else _n_global
        self.row_begin = _row_begin
        self.jitter_factor = jitter_factor
        self.precision = precision_code(precision)
        self._keep = []
        self.m = None
        self._h = None
        self._data = (x_or_mu, s, y, on_dev)

    def _create(self, m: int):
        cfg = L.engine_config(int(self.kind), self.n_global, self.row_begin, self.n, self.q, self.d, m,
                              self.jitter_factor, self.precision)
        h = C.c_void_p()
        check(self._lib.sgpx_engine_create(self.ctx.handle, C.byref(cfg), C.byref(h)))
        self._h = h
        self.m = m
        self._grads_registered = False
        x, s, y, on_dev = self._data
        if on_dev:
            xv = device_view(x)
            sv = device_view(s) if self.kind == ModelKind.latent else L.cmat(None, 0, 0, 0)
            yv = device_view(y)
            self._keep = [x, s, y]
        else:
            xa, ya = _F(x), _F(y)
            sa = _F(s) if self.kind == ModelKind.latent else _EMPTY
            xv, sv, yv = _cm(xa), _cm(sa), _cm(ya)
            self._keep = [xa, sa, ya]
        check(self._lib.sgpx_engine_set_data(self._h, xv, sv, yv, 1 if on_dev else 0))

    def broadcast(self, kernel: KernelSpec, beta: float, z, mu=None, s=None):
        """Engine::broadcast (parallel.hpp:358-367)."""
        z = _F(z)
        if self._h is None:
            self._create(z.shape[0])
        if z.shape[0] != self.m:
            raise SgpxInvalidArgument("broadcast: Z must keep M rows for the engine's lifetime")
        ks = kernel._c()
        self._kernel = kernel
        self._z = z
        nullm = L.cmat(None, 0, 0, 0)
        if mu is not None and _is_cuda_tensor(mu):
            self._keep_local = [mu, s]
            check(self._lib.sgpx_engine_broadcast(self._h, C.byref(ks), float(beta), _cm(z), device_view(mu),
                                                  device_view(s), 1))
        elif mu is not None:
            ma, sa = _F(mu), _F(s)
            self._keep_local = [ma, sa]
            check(self._lib.sgpx_engine_broadcast(self._h, C.byref(ks), float(beta), _cm(z), _cm(ma), _cm(sa), 0))
        else:
            check(self._lib.sgpx_engine_broadcast(self._h, C.byref(ks), float(beta), _cm(z), nullm, nullm, 0))
        self.beta = beta

    def _result_buffers(self):
        m, d, q = self.m, self.d, self.q
        bufs = dict(psi_y=np.zeros((m, d), order="F"), phi_big=np.zeros((m, m), order="F"),
                    d_z=np.zeros((m, q), order="F"), d_ls=np.zeros(q))
        r = L.eval_result()
        r.psi_y = bufs["psi_y"].ctypes.data_as(C.c_void_p)
        r.phi_big = bufs["phi_big"].ctypes.data_as(C.c_void_p)
        r.d_z = bufs["d_z"].ctypes.data_as(C.c_void_p)
        r.d_lengthscales = bufs["d_ls"].ctypes.data_as(C.c_void_p)
        return r, bufs

    def set_local_grads_out(self, dmu, ds):
        """Preallocated host buffers (pinned for overlap) that evaluate() fills with d_mu / d_s.
        The engine streams them per sub-shard while the rest of the gradient pass computes
        (sgpx_engine_set_local_grads_out); ``None`` unregisters."""
        if dmu is None:
            self._grads_out = None
            if self._h is not None:
                nm = L.mmat(None, 0, 0, 0)
                check(self._lib.sgpx_engine_set_local_grads_out(self._h, nm, nm))
            return
        n, q = self.n, self.q
        for a in (dmu, ds):
            if a.shape != (n, q) or a.dtype != np.float64 or not a.flags.f_contiguous:
                raise SgpxInvalidArgument("local grads out: Fortran-ordered float64 n_local x Q arrays required")
        self._grads_out = (dmu, ds)
        self._grads_registered = False

    def _register_grads_out(self):
        if getattr(self, "_grads_out", None) is not None and not getattr(self, "_grads_registered", False) \
                and self._h is not None:
            dmu, ds = self._grads_out
            check(self._lib.sgpx_engine_set_local_grads_out(self._h, _cm(dmu), _cm(ds)))
            self._grads_registered = True

    def _pack(self, r, bufs, with_grads, local_to_host=True) -> EvalResult:
        stats = SufficientStats(r.phi, bufs["psi_y"], bufs["phi_big"], r.yy, int(r.n_count))
        g = GradientParts()
        if with_grads:
            g.d_z = bufs["d_z"]
            g.d_lengthscales = bufs["d_ls"]
            g.d_variance = r.d_variance
            g.d_beta = r.d_beta
            if self.kind == ModelKind.latent and local_to_host:
                if getattr(self, "_grads_registered", False):
                    g.d_mu, g.d_s = self._grads_out  # streamed by the engine during evaluate()
                else:
                    g.d_mu, g.d_s = self.local_grads(getattr(self, "_grads_out", None))
        t = EngineTimings(r.stats_pass_s, r.coordinator_s, r.grad_pass_s, r.wall_s, r.fwd_kernel_s, r.bwd_kernel_s,
                          r.fwd_grid, r.bwd_grid, L.PRECISION_NAMES.get(int(r.precision_used), "none"),
                          float(r.z_spread), float(r.psi2_fwd_kernel_s), float(r.psi2_bwd_kernel_s))
        return EvalResult(BoundBreakdown._from(r.bound), stats, bool(r.has_grads), g, t, r.jitter_factor_used)

    def evaluate(self, with_grads: bool = True, local_to_host: bool = True) -> EvalResult:
        """Engine::evaluate (parallel.hpp:370-450)."""
        r, bufs = self._result_buffers()
        if local_to_host and with_grads and self.kind == ModelKind.latent:
            self._register_grads_out()
        elif getattr(self, "_grads_registered", False):  # device-only evaluation: do not stream
            nm = L.mmat(None, 0, 0, 0)
            check(self._lib.sgpx_engine_set_local_grads_out(self._h, nm, nm))
            self._grads_registered = False
        check(self._lib.sgpx_engine_evaluate(self._h, 1 if with_grads else 0, C.byref(r)))
        return self._pack(r, bufs, with_grads, local_to_host)

    def local_grads(self, out=None):
        """(d_mu, d_s) on the host, n_local x Q.  ``out``: optional preallocated Fortran-ordered
        float64 pair (e.g. views of pinned memory) to avoid a pageable copy."""
        n, q = self.n, self.q
        if out is None:
            dmu = np.zeros((n, q), order="F")
            ds = np.zeros((n, q), order="F")
        else:
            dmu, ds = out
            if not (dmu.flags.f_contiguous and ds.flags.f_contiguous and dmu.shape == (n, q) == ds.shape):
                raise SgpxInvalidArgument("local_grads out= must be two Fortran-ordered n_local x Q arrays")
        check(self._lib.sgpx_engine_copy_local_grads(self._h, _cm(dmu), _cm(ds)))
        return dmu, ds

    def finalize(self):
        """The reference's finalize(): an evaluation (bound only) at the current parameters, whose
        factors predict() serves from; returns the cached bound."""
        return self.evaluate(False).bound.total

    def predict(self, x_star, mode: str = "observation"):
        """predict_from_cache (model.hpp:197-217): (mean T x D, variance T x D) at the rows of x_star
        (latent points for the GP-LVM); ``mode`` "observation" adds the 1/beta noise, "latent" does not."""
        if mode not in ("observation", "latent"):
            raise SgpxInvalidArgument("predict: mode must be 'observation' or 'latent'")
        if self._h is None:
            raise SgpxInvalidArgument("predict() before fit()/finalize()")
        xs = _F(x_star)
        t = xs.shape[0]
        mean = np.zeros((t, self.d), order="F")
        var = np.zeros((t, self.d), order="F")
        cb = C.c_double()
        check(self._lib.sgpx_engine_predict(self._h, _cm(xs), 1 if mode == "observation" else 0, _cm(mean),
                                            _cm(var), C.byref(cb)))
        self.cached_bound = cb.value
        return mean, var

    def local_grads_device(self):
        """(d_mu, d_s) device pointers, n x Q column-major fp64."""
        a, b = C.c_void_p(), C.c_void_p()
        check(self._lib.sgpx_engine_local_grads_device(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def close(self):
        if self._h is not None:
            self._lib.sgpx_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class LbfgsOptions:
    """LbfgsOptions (optimizer.hpp:154-163)."""
    memory: int = 10
    c1: float = 1e-4
    c2: float = 0.9
    g_tol: float = 1e-5
    f_tol: float = 1e-9
    max_iters: int = 500
    max_evals: int = 0
    max_line_search: int = 40

    def _c(self):
        return L.lbfgs_options(self.memory, self.c1, self.c2, self.g_tol, self.f_tol, self.max_iters,
                               self.max_evals, self.max_line_search)


class FitSession:
    """FitSession (model.hpp:100-168): the engine, the packed parameters and the stepwise L-BFGS state,
    with the parameter vector and the L-BFGS history resident on the GPU (sgpx_fit_*).
    ``step()`` is one sync_step; ``bound`` = -value; ``params()`` unpacks the current iterate."""

    def __init__(self, kind, x_or_mu, s, y, kernel: KernelSpec, beta: float, z, options: LbfgsOptions | None = None,
                 precision: str = "auto", ctx: Context | None = None):
        self.kind = ModelKind(kind)
        latent = self.kind == ModelKind.latent
        self.engine = Engine(kind, x_or_mu, s, y, ctx=ctx, precision=precision)
        z = _F(z)
        self.engine._create(z.shape[0])
        self.options = options or LbfgsOptions()
        self._lib = L.load()
        self.q, self.m, self.n = z.shape[1], z.shape[0], self.engine.n
        ks = kernel._c()
        mu_c = _cm(_F(x_or_mu)) if latent else L.cmat(None, 0, 0, 0)
        s_c = _cm(_F(s)) if latent else L.cmat(None, 0, 0, 0)
        self._keep = (x_or_mu, s)
        h = C.c_void_p()
        oc = self.options._c()
        rc = self._lib.sgpx_fit_create(self.engine._h, self.n, C.byref(ks), float(beta), _cm(z), mu_c, s_c,
                                       C.byref(oc), C.byref(h))
        self._check(rc)
        self._h = h

    def _check(self, rc):
        if rc != L.SGPX_OK:
            msg = self._lib.sgpx_fit_last_error().decode(errors="replace")
            raise (SgpxNumericError if rc == L.SGPX_NUMERIC else SgpxError)(msg)

    def step(self) -> bool:
        adv = C.c_int()
        self._check(self._lib.sgpx_fit_step(self._h, C.byref(adv)))
        return bool(adv.value)

    def state(self) -> dict:
        v, gn = C.c_double(), C.c_double()
        it, ev, le, st = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        self._check(self._lib.sgpx_fit_state(self._h, C.byref(v), C.byref(gn), C.byref(it), C.byref(ev), C.byref(le),
                                             C.byref(st)))
        return dict(value=v.value, bound=-v.value, grad_norm=gn.value, iterations=it.value, total_evals=ev.value,
                    last_step_evals=le.value, status=L.FIT_STATUS.get(st.value, "unknown"),
                    message=self._lib.sgpx_fit_message(self._h).decode())

    def params(self) -> dict:
        var, beta = C.c_double(), C.c_double()
        ls = np.zeros(self.q)
        z = np.zeros((self.m, self.q), order="F")
        latent = self.kind == ModelKind.latent
        mu = np.zeros((self.n, self.q), order="F") if latent else None
        s = np.zeros((self.n, self.q), order="F") if latent else None
        nm = L.mmat(None, 0, 0, 0)
        self._check(self._lib.sgpx_fit_params(self._h, C.byref(var), ls.ctypes.data_as(C.c_void_p), C.byref(beta),
                                              _cm(z), _cm(mu) if latent else nm, _cm(s) if latent else nm))
        return dict(variance=var.value, lengthscales=ls, beta=beta.value, z=z, mu=mu, s=s)

    def close(self):
        if getattr(self, "_h", None) is not None:
            self._lib.sgpx_fit_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MultiEngine:
    """sgp::Engine(kind, x, s, y, workers) over several GPUs of one process (sgpx_multi_*): shards by
    make_partition, shard i on ``devices[i]`` (default: round-robin over the visible GPUs), the two
    exchanges folded per device and allreduced with NCCL across devices."""

    def __init__(self, kind, x_or_mu, s, y, workers: int, tiles: TileConfig | None = None,
                 jitter_factor: float = 1e-6, devices=None, precision: str = "auto"):
        self.kind = ModelKind(kind)
        (tiles or TileConfig())
        self._lib = L.load()
        x = _F(x_or_mu)
        y = _F(y)
        s = _F(s) if self.kind == ModelKind.latent else _EMPTY
        self.n, self.q = x.shape
        self.d = y.shape[1]
        self.workers = int(workers)
        if devices is None:
            nd = max(1, device_count())
            devices = [i % nd for i in range(self.workers)]
        self.devices = (C.c_int * self.workers)(*devices)
        self.jitter_factor = jitter_factor
        self.precision = precision_code(precision)
        self._data = (x, s, y)
        self._h = None
        self.m = None

    def _create(self, m):
        cfg = L.engine_config(int(self.kind), self.n, 0, self.n, self.q, self.d, m, self.jitter_factor,
                              self.precision)
        h = C.c_void_p()
        check(self._lib.sgpx_multi_create(self.workers, self.devices, C.byref(cfg), C.byref(h)))
        self._h = h
        self.m = m
        x, s, y = self._data
        check(self._lib.sgpx_multi_set_data(self._h, _cm(x), _cm(s), _cm(y)))

    def broadcast(self, kernel: KernelSpec, beta: float, z, mu=None, s=None):
        z = _F(z)
        if self._h is None:
            self._create(z.shape[0])
        ks = kernel._c()
        nullm = L.cmat(None, 0, 0, 0)
        if mu is not None:
            self._local = (_F(mu), _F(s))
            check(self._lib.sgpx_multi_broadcast(self._h, C.byref(ks), float(beta), _cm(z), _cm(self._local[0]),
                                                 _cm(self._local[1])))
        else:
            check(self._lib.sgpx_multi_broadcast(self._h, C.byref(ks), float(beta), _cm(z), nullm, nullm))
        self.beta = beta

    def evaluate(self, with_grads: bool = True) -> EvalResult:
        m, d, q, n = self.m, self.d, self.q, self.n
        bufs = dict(psi_y=np.zeros((m, d), order="F"), phi_big=np.zeros((m, m), order="F"),
                    d_z=np.zeros((m, q), order="F"), d_ls=np.zeros(q))
        r = L.eval_result()
        r.psi_y = bufs["psi_y"].ctypes.data_as(C.c_void_p)
        r.phi_big = bufs["phi_big"].ctypes.data_as(C.c_void_p)
        r.d_z = bufs["d_z"].ctypes.data_as(C.c_void_p)
        r.d_lengthscales = bufs["d_ls"].ctypes.data_as(C.c_void_p)
        latent = self.kind == ModelKind.latent
        dmu = np.zeros((n, q), order="F") if latent else None
        ds = np.zeros((n, q), order="F") if latent else None
        nullm = L.mmat(None, 0, 0, 0)
        check(self._lib.sgpx_multi_evaluate(self._h, 1 if with_grads else 0, C.byref(r),
                                            _cm(dmu) if latent else nullm, _cm(ds) if latent else nullm))
        stats = SufficientStats(r.phi, bufs["psi_y"], bufs["phi_big"], r.yy, int(r.n_count))
        g = GradientParts()
        if with_grads:
            g.d_z, g.d_lengthscales, g.d_variance, g.d_beta = bufs["d_z"], bufs["d_ls"], r.d_variance, r.d_beta
            g.d_mu, g.d_s = dmu, ds
        t = EngineTimings(r.stats_pass_s, r.coordinator_s, r.grad_pass_s, r.wall_s, r.fwd_kernel_s, r.bwd_kernel_s,
                          r.fwd_grid, r.bwd_grid, L.PRECISION_NAMES.get(int(r.precision_used), "none"),
                          float(r.z_spread), float(r.psi2_fwd_kernel_s), float(r.psi2_bwd_kernel_s))
        return EvalResult(BoundBreakdown._from(r.bound), stats, bool(r.has_grads), g, t, r.jitter_factor_used)

    def close(self):
        if self._h is not None:
            self._lib.sgpx_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# coordinator (host fp64; used by the multi-rank engine and its CPU tests)
# ---------------------------------------------------------------------------
def packed_stats_count(m: int, d: int) -> int:
    return 4 + m * (m + 1) // 2 + m * d


def packed_grads_count(m: int, q: int) -> int:
    return 1 + q + m * q


def pack_stats(phi, yy, n, kl, phi_big, psi_y) -> np.ndarray:
    """Allreduce #1 payload layout (sgpx.h)."""
    m = phi_big.shape[0]
    iu = np.triu_indices(m)
    # m1-major upper triangle == row-major traversal of (a, b>=a)
    return np.concatenate([[phi, yy, n, kl], np.asarray(phi_big)[iu], _F(psi_y).ravel(order="F")])


def coordinate_host(kind, n, d, packed_stats, z, kernel: KernelSpec, beta, jitter_factor=1e-6, adjoints=True):
    z = _F(z)
    m = z.shape[0]
    ps = np.ascontiguousarray(packed_stats, dtype=np.float64)
    bd = L.bound_breakdown()
    sc = np.zeros(3)
    dpsi = np.zeros((m, d), order="F")
    dphi = np.zeros((m, m), order="F")
    dk = np.zeros((m, m), order="F")
    ks = kernel._c()
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    check(L.load().sgpx_coordinate_host(int(kind), n, d, m, p(ps), _cm(z), C.byref(ks), float(beta),
                                        float(jitter_factor), C.byref(bd), p(sc) if adjoints else None, p(dpsi),
                                        p(dphi), p(dk)))
    out = dict(bound=BoundBreakdown._from(bd))
    if adjoints:
        out.update(d_phi=sc[0], d_beta=sc[1], jitter_factor=sc[2], d_psi_y=dpsi, d_phi_big=dphi, d_kmm=dk)
    return out


def finish_host(packed_grads, z, kernel: KernelSpec, d_kmm, jitter_factor):
    z = _F(z)
    m, q = z.shape
    pg = np.ascontiguousarray(packed_grads, dtype=np.float64)
    dk = _F(d_kmm)
    dz = np.zeros((m, q), order="F")
    dls = np.zeros(q)
    dv = C.c_double()
    ks = kernel._c()
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    check(L.load().sgpx_finish_host(m, q, p(pg), _cm(z), C.byref(ks), p(dk), float(jitter_factor), p(dz),
                                    C.byref(dv), p(dls)))
    return dz, dv.value, dls


# ---------------------------------------------------------------------------
# seeded inputs and binary matrices (common.hpp:45-97, model.hpp:420-429, io.hpp:114-153)
# ---------------------------------------------------------------------------
def rng_normal_matrix(seed: int, rows: int, cols: int, device=None, ctx: Context | None = None):
    """Rng(seed).normal_matrix(rows, cols), generated on the GPU.  ``device``: return a column-major
    CUDA float64 tensor there (the data never visits the host); else a Fortran-ordered numpy array."""
    ctx = ctx or Context.default()
    lib = L.load()
    if device is not None:
        import torch

        t = torch.empty((cols, rows), dtype=torch.float64, device=device).t()
        v = device_view(t) if rows * cols else L.cmat(None, rows, cols, max(rows, 1))
        check(lib.sgpx_rng_normal_matrix(ctx.handle, C.c_uint64(seed), rows, cols, v, 1))
        return t
    out = np.zeros((rows, cols), order="F")
    check(lib.sgpx_rng_normal_matrix(ctx.handle, C.c_uint64(seed), rows, cols, _cm(out), 0))
    return out


def rng_choose_rows(seed: int, n: int, m: int) -> np.ndarray:
    """The M distinct rows init_gplvm takes for Z (partial Fisher-Yates with Rng(seed))."""
    idx = np.zeros(m, dtype=np.int64)
    check(L.load().sgpx_rng_choose_rows(C.c_uint64(seed), n, m, idx.ctypes.data_as(C.c_void_p)))
    return idx


def write_matrix_bin(base: str, a):
    """write_matrix_bin (io.hpp:119-132): <base>.shape + row-major float64 <base>.bin."""
    a = _F(a)
    check(L.load().sgpx_io_write_matrix(str(base).encode(), _cm(a)))


def read_matrix_bin(base: str) -> np.ndarray:
    """read_matrix_bin (io.hpp:134-153)."""
    r, c = C.c_int64(), C.c_int64()
    lib = L.load()
    check(lib.sgpx_io_matrix_shape(str(base).encode(), C.byref(r), C.byref(c)))
    out = np.zeros((r.value, c.value), order="F")
    check(lib.sgpx_io_read_matrix(str(base).encode(), _cm(out)))
    return out


def load_matrix_bin_device(base: str, device="cuda", ctx: Context | None = None):
    """read_matrix_bin straight into a column-major CUDA tensor (pinned slabs + device transpose)."""
    import torch

    ctx = ctx or Context.default()
    lib = L.load()
    r, c = C.c_int64(), C.c_int64()
    check(lib.sgpx_io_matrix_shape(str(base).encode(), C.byref(r), C.byref(c)))
    t = torch.empty((c.value, r.value), dtype=torch.float64, device=device).t()
    v = device_view(t) if r.value * c.value else L.cmat(None, r.value, c.value, max(r.value, 1))
    check(lib.sgpx_io_load_matrix_device(ctx.handle, str(base).encode(), v))
    return t
