"""CPU ORACLE — test infrastructure only.

ctypes bindings over ``oracle/liboracle.so`` (built from ``oracle/sgp_oracle.cpp``,
a plain-C++ fp64 restatement of the reference hot path; see that file's header
for the reference file:line map).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (cpu_baseline leg and ``--impl reference``) may import this
package, and only as the checker / CPU baseline.  The product package
``paper_1410_4984_b200`` never imports it.

Arrays are numpy float64, column-major (Fortran order) like Eigen::MatrixXd.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
# CPU-baseline build of the same source: -ffast-math lets g++ vectorise the exp loops through glibc's
# libmvec (AVX2 _ZGVdN4v_exp) and the tile sums, the way Eigen's packet math evaluates the reference's
# array expressions.  Timing only; the checker is always the strict build.
SIMD_LIB_PATH = os.path.join(_HERE, "liboracle_simd.so")
SRC_PATH = os.path.join(_HERE, "sgp_oracle.cpp")

_lib = None
_simd_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle restatement (g++, portable x86-64-v3 so it runs on the GPU box host), strict
    and SIMD-baseline builds."""
    for path, extra in ((LIB_PATH, []), (SIMD_LIB_PATH, ["-ffast-math"])):
        if force or not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(SRC_PATH):
            cmd = ["g++", "-std=c++17", "-O3", "-march=x86-64-v3", *extra, "-fPIC", "-shared", "-pthread",
                   "-o", path, SRC_PATH]
            subprocess.check_call(cmd)
    return LIB_PATH


def _load(path):
    lb = C.CDLL(path)
    lb.oracle_last_error.restype = C.c_char_p
    lb.oracle_rng_normal_matrix.restype = None
    lb.oracle_rng_uniform.restype = None
    lb.oracle_rng_choose_rows.restype = None
    return lb


def lib(simd: bool = False):
    global _lib, _simd_lib
    if simd:
        if _simd_lib is None:
            build()
            _simd_lib = _load(SIMD_LIB_PATH)
        return _simd_lib
    if _lib is None:
        build()
        _lib = _load(LIB_PATH)
    return _lib


class OracleError(Exception):
    pass


class OracleInvalidArgument(OracleError, ValueError):
    pass


class OracleNumericError(OracleError, ArithmeticError):
    pass


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().oracle_last_error().decode()
    if rc == 1:
        raise OracleInvalidArgument(msg)
    if rc == 2:
        raise OracleNumericError(msg)
    raise OracleError(msg)


def F(a) -> np.ndarray:
    """Column-major float64 copy/view."""
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _i64(x):
    return C.c_int64(int(x))


def _d(x):
    return C.c_double(float(x))


@dataclass
class Stats:
    phi: float
    yy: float
    n_count: int
    psi_y: np.ndarray
    phi_big: np.ndarray


@dataclass
class Grads:
    d_mu: np.ndarray | None
    d_s: np.ndarray | None
    d_z: np.ndarray
    d_variance: float
    d_lengthscales: np.ndarray


def sweep_stats(expected, mu, s, y, z, variance, lengthscales, adj=None, grads=False,
                block_span=64, thread_span=1024):
    """Restatement of sgp::detail::sweep_stats (psi_stats.hpp:108-326).

    adj: None or (d_phi, d_psi_y[M,D], d_phi_big[M,M]).  Returns (Stats, Grads|None).
    """
    mu = F(mu)
    y = F(y)
    z = F(z)
    n, q = mu.shape
    m = z.shape[0]
    d = y.shape[1]
    s = F(s) if expected else None
    ls = F(np.broadcast_to(np.asarray(lengthscales, dtype=np.float64), (q,)))
    scal = np.zeros(3)
    psi_y = np.zeros((m, d), order="F")
    phi_big = np.zeros((m, m), order="F")
    has_adj = adj is not None
    d_phi, d_psi_y, d_phi_big = (0.0, np.zeros((m, d), order="F"), np.zeros((m, m), order="F"))
    if has_adj:
        d_phi, d_psi_y, d_phi_big = adj
        d_psi_y, d_phi_big = F(d_psi_y), F(d_phi_big)
    want = grads or has_adj
    g_mu = np.zeros((n, q), order="F") if want else None
    g_s = np.zeros((n, q), order="F") if want else None
    g_z = np.zeros((m, q), order="F") if want else None
    g_var = np.zeros(1)
    g_ls = np.zeros(q)
    rc = lib().oracle_sweep_stats(
        C.c_int(1 if expected else 0), _i64(n), _i64(q), _i64(m), _i64(d), _p(mu), _p(s), _p(y), _p(z),
        _d(variance), _p(ls), _i64(block_span), _i64(thread_span), C.c_int(1 if has_adj else 0), _d(d_phi),
        _p(d_psi_y), _p(d_phi_big), _p(scal), _p(psi_y), _p(phi_big), _p(g_mu), _p(g_s), _p(g_z),
        _p(g_var), _p(g_ls))
    _check(rc)
    st = Stats(scal[0], scal[1], int(scal[2]), psi_y, phi_big)
    if not want:
        return st, None
    return st, Grads(g_mu if expected else None, g_s if expected else None, g_z, float(g_var[0]), g_ls)


def psi1_expected(mu, s, z, variance, lengthscales):
    mu, s, z = F(mu), F(s), F(z)
    n, q = mu.shape
    m = z.shape[0]
    ls = F(np.broadcast_to(np.asarray(lengthscales, dtype=np.float64), (q,)))
    out = np.zeros((n, m), order="F")
    _check(lib().oracle_psi1_expected(_i64(n), _i64(q), _i64(m), _p(mu), _p(s), _p(z), _d(variance), _p(ls),
                                      _p(out)))
    return out


def kern_cross(x, z, variance, lengthscales):
    x, z = F(x), F(z)
    n, q = x.shape
    m = z.shape[0]
    ls = F(np.broadcast_to(np.asarray(lengthscales, dtype=np.float64), (q,)))
    out = np.zeros((n, m), order="F")
    _check(lib().oracle_kern_cross(_i64(n), _i64(m), _i64(q), _p(x), _p(z), _d(variance), _p(ls), _p(out)))
    return out


def kern_gram(z, variance, lengthscales, jitter):
    z = F(z)
    m, q = z.shape
    ls = F(np.broadcast_to(np.asarray(lengthscales, dtype=np.float64), (q,)))
    out = np.zeros((m, m), order="F")
    dup = C.c_int(0)
    _check(lib().oracle_kern_gram(_i64(m), _i64(q), _p(z), _d(variance), _p(ls), _d(jitter), _p(out),
                                  C.byref(dup)))
    return out, bool(dup.value)


def kern_grads(x, z, variance, lengthscales, upstream):
    x, z, up = F(x), F(z), F(upstream)
    n, q = x.shape
    m = z.shape[0]
    ls = F(np.broadcast_to(np.asarray(lengthscales, dtype=np.float64), (q,)))
    dv = np.zeros(1)
    dls = np.zeros(q)
    dz = np.zeros((m, q), order="F")
    dx = np.zeros((n, q), order="F")
    _check(lib().oracle_kern_grads(_i64(n), _i64(m), _i64(q), _p(x), _p(z), _d(variance), _p(ls), _p(up),
                                   _p(dv), _p(dls), _p(dz), _p(dx)))
    return dict(d_variance=float(dv[0]), d_lengthscales=dls, d_z=dz, d_x=dx)


def factor_gram(z, variance, lengthscales, jitter_factor=1e-6):
    z = F(z)
    m, q = z.shape
    ls = F(np.broadcast_to(np.asarray(lengthscales, dtype=np.float64), (q,)))
    kmm = np.zeros((m, m), order="F")
    out = np.zeros(3)
    _check(lib().oracle_factor_gram(_i64(m), _i64(q), _p(z), _d(variance), _p(ls), _d(jitter_factor), _p(kmm),
                                    _p(out[0:1]), _p(out[1:2]), _p(out[2:3])))
    return dict(kmm=kmm, jitter=out[0], jitter_factor=out[1], log_det=out[2])


BOUND_FIELDS = ("total", "log_det_term", "data_fit_term", "quadratic_term", "trace_phi_term",
                "trace_kmm_term", "kl_term")


def bound(stats: Stats, kmm, beta, n, d, adjoints=True):
    """bound_core + adjoints_from_core (bound.hpp:84-119, 196-226)."""
    m = kmm.shape[0]
    bd = np.zeros(7)
    sc = np.zeros(2)
    dpsi = np.zeros((m, d), order="F")
    dphi = np.zeros((m, m), order="F")
    dk = np.zeros((m, m), order="F")
    _check(lib().oracle_bound(_i64(m), _i64(d), _i64(n), _d(stats.phi), _d(stats.yy), _p(F(stats.psi_y)),
                              _p(F(stats.phi_big)), _p(F(kmm)), _d(beta), _p(bd),
                              _p(sc) if adjoints else None, _p(dpsi), _p(dphi), _p(dk)))
    out = dict(zip(BOUND_FIELDS, bd))
    if adjoints:
        out.update(d_phi=sc[0], d_beta=sc[1], d_psi_y=dpsi, d_phi_big=dphi, d_kmm=dk)
    return out


@dataclass
class EvalResult:
    bound: dict
    stats: Stats
    d_mu: np.ndarray | None = None
    d_s: np.ndarray | None = None
    d_z: np.ndarray | None = None
    d_variance: float = 0.0
    d_beta: float = 0.0
    d_lengthscales: np.ndarray | None = None
    wall_s: float = 0.0
    coordinator_s: float = 0.0


def engine_evaluate(latent, x_or_mu, s, y, z, variance, lengthscales, beta, workers=1, with_grads=True,
                    block_span=64, thread_span=1024, jitter_factor=1e-6, simd=False) -> EvalResult:
    """Restatement of Engine(kind, ...).evaluate(with_grads) (parallel.hpp:370-450).  ``simd``: the
    vectorised CPU-baseline build (timing), else the strict checker."""
    x = F(x_or_mu)
    y = F(y)
    z = F(z)
    n, q = x.shape
    d = y.shape[1]
    m = z.shape[0]
    s = F(s) if latent else None
    ls = F(np.broadcast_to(np.asarray(lengthscales, dtype=np.float64), (q,)))
    bd = np.zeros(7)
    sc = np.zeros(3)
    psi_y = np.zeros((m, d), order="F")
    phi_big = np.zeros((m, m), order="F")
    d_mu = np.zeros((n, q), order="F")
    d_s = np.zeros((n, q), order="F")
    d_z = np.zeros((m, q), order="F")
    gs = np.zeros(2)
    dls = np.zeros(q)
    times = np.zeros(2)
    _check(lib(simd).oracle_engine_evaluate(
        C.c_int(1 if latent else 0), _i64(n), _i64(q), _i64(d), _i64(m), _p(x), _p(s), _p(y), _p(z),
        _d(variance), _p(ls), _d(beta), C.c_int(workers), _i64(block_span), _i64(thread_span), _d(jitter_factor),
        C.c_int(1 if with_grads else 0), _p(bd), _p(sc), _p(psi_y), _p(phi_big), _p(d_mu), _p(d_s), _p(d_z),
        _p(gs), _p(dls), _p(times)))
    res = EvalResult(dict(zip(BOUND_FIELDS, bd)), Stats(sc[0], sc[1], int(sc[2]), psi_y, phi_big),
                     wall_s=times[0], coordinator_s=times[1])
    if with_grads:
        res.d_mu = d_mu if latent else None
        res.d_s = d_s if latent else None
        res.d_z = d_z
        res.d_variance = gs[0]
        res.d_beta = gs[1]
        res.d_lengthscales = dls
    return res


def predict(latent, x_or_mu, s, y, z, variance, lengthscales, beta, x_star, observation=True, jitter_factor=1e-6):
    """finalize() + predict(X*) of SparseGPRegression / BayesianGPLVM (model.hpp:181-217, 265-296, 353-383):
    returns (mean T x D, variance T x D, cached_bound)."""
    x = F(x_or_mu)
    y = F(y)
    z = F(z)
    xs = F(x_star)
    n, q = x.shape
    d = y.shape[1]
    m = z.shape[0]
    t = xs.shape[0]
    s = F(s) if latent else None
    ls = F(np.broadcast_to(np.asarray(lengthscales, dtype=np.float64), (q,)))
    mean = np.zeros((t, d), order="F")
    var = np.zeros((t, d), order="F")
    bound = C.c_double()
    _check(lib().oracle_predict(C.c_int(1 if latent else 0), _i64(n), _i64(q), _i64(d), _i64(m), _p(x), _p(s), _p(y),
                                _p(z), _d(variance), _p(ls), _d(beta), _d(jitter_factor), _i64(t), _p(xs),
                                C.c_int(1 if observation else 0), _p(mean), _p(var), C.byref(bound)))
    return mean, var, bound.value


def fit(latent, x_or_mu, s, y, z, variance, lengthscales, beta, iters, workers=1):
    """FitSession + LbfgsState (model.hpp:100-168, optimizer.hpp:20-458) on the oracle engine: `iters`
    sync_steps.  Returns dict(values=-bound per accepted iterate, grad_norms, status, evals, params)."""
    x = F(x_or_mu)
    y = F(y)
    z = F(z)
    n, q = x.shape
    d = y.shape[1]
    m = z.shape[0]
    s = F(s) if latent else None
    ls = F(np.broadcast_to(np.asarray(lengthscales, dtype=np.float64), (q,)))
    values = np.full(iters + 1, np.nan)
    gnorms = np.full(iters + 1, np.nan)
    status, evals = C.c_int(), C.c_int()
    var_o, beta_o = C.c_double(), C.c_double()
    ls_o = np.zeros(q)
    z_o = np.zeros((m, q), order="F")
    mu_o = np.zeros((n, q), order="F") if latent else None
    s_o = np.zeros((n, q), order="F") if latent else None
    _check(lib().oracle_fit(C.c_int(1 if latent else 0), _i64(n), _i64(q), _i64(d), _i64(m), _p(x), _p(s), _p(y),
                            _p(z), _d(variance), _p(ls), _d(beta), C.c_int(workers), C.c_int(iters), _p(values),
                            _p(gnorms), C.byref(status), C.byref(evals), C.byref(var_o), _p(ls_o), C.byref(beta_o),
                            _p(z_o), _p(mu_o), _p(s_o)))
    return dict(values=values, grad_norms=gnorms, status=status.value, evals=evals.value,
                params=dict(variance=var_o.value, lengthscales=ls_o, beta=beta_o.value, z=z_o, mu=mu_o, s=s_o))


def rng_normal_matrix(seed, rows, cols):
    """Rng(seed).normal_matrix(rows, cols) (common.hpp:86-91), column-major result."""
    out = np.zeros((rows, cols), order="F")
    lib().oracle_rng_normal_matrix(C.c_uint64(seed), _i64(rows), _i64(cols), _p(out))
    return out


def rng_choose_rows(seed, n, m):
    """init_gplvm's M distinct Z rows (model.hpp:420-429, partial Fisher-Yates with Rng(seed))."""
    out = np.zeros(m, dtype=np.int64)
    lib().oracle_rng_choose_rows(C.c_uint64(seed), _i64(n), _i64(m), out.ctypes.data_as(C.c_void_p))
    return out


def rng_uniform(seed, count):
    out = np.zeros(count)
    lib().oracle_rng_uniform(C.c_uint64(seed), _i64(count), _p(out))
    return out


def make_partition(n, p):
    b = np.zeros(p, dtype=np.int64)
    e = np.zeros(p, dtype=np.int64)
    _check(lib().oracle_make_partition(_i64(n), C.c_int(p), _p(b), _p(e)))
    return list(zip(b.tolist(), e.tolist()))
