"""Accuracy envelope of the row-tile path, per element (the reference's rel_err, oracles.hpp:55-58:
|a-b| / max(|a|, |b|, 1)) and norm-wise, against the fp64 oracle, for data layouts that stress
the exponent-as-GEMM expansion: Gaussian spreads, a bimodal Z, a far cluster without inducing
points, a handful of far outlier rows.  Prints the spread statistics the precision decision
sees (Tz = max_a sum_q ((z_a - c) / l)^2, Tx = max_n sum_q ((mu_n - c) / l)^2 / t_nq) next to
the errors.  Usage: SGPX_PSI_MODE=fast|precise|direct python tools/envelope.py [case ...]
(a case prefixed det- runs the deterministic / SGPR mode on the same X = mu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1410_4984_b200 import sgp  # noqa: E402

oracle.lib()


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    sc = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)
    return float(np.max(np.abs(a - b) / sc)) if a.size else 0.0


def nre(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def case(name, n=4000, q=10, d=10, m=100, seed=1):
    expected = not name.startswith("det-")
    name0 = name
    name = name[4:] if not expected else name
    rng = np.random.default_rng(seed)
    s = rng.uniform(0.25, 1.0, (n, q))
    y = rng.normal(size=(n, d))
    ls = rng.uniform(0.5, 2.0, q)
    kind, _, arg = name.partition(":")
    f = float(arg) if arg else 1.0
    if kind == "gauss":  # mu ~ N(0, f^2), Z from mu
        mu = f * rng.normal(size=(n, q))
        z = mu[rng.choice(n, m, replace=False)] + 0.05 * rng.normal(size=(m, q))
    elif kind == "bimodal":  # two clusters at +-f l (dimension 0), inducing points in both
        mu = rng.normal(size=(n, q))
        sign = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
        mu[:, 0] += sign * f * ls[0]
        z = mu[rng.choice(n, m, replace=False)] + 0.05 * rng.normal(size=(m, q))
    elif kind == "farcluster":  # 10 % of the rows at f l, no inducing point there
        mu = rng.normal(size=(n, q))
        z = mu[rng.choice(n, m, replace=False)] + 0.05 * rng.normal(size=(m, q))
        mu[: n // 10, 0] += f * ls[0]
    elif kind == "outliers":  # 8 rows at f l along every dimension, Z from the bulk
        mu = rng.normal(size=(n, q))
        z = mu[rng.choice(np.arange(8, n), m, replace=False)] + 0.05 * rng.normal(size=(m, q))
        mu[:8] += f * ls
    elif kind == "zcluster":  # a small far cluster (5 % of rows) holding 5 inducing points
        mu = rng.normal(size=(n, q))
        k = n // 20
        mu[:k, 0] += f * ls[0]
        idx = np.concatenate([rng.choice(k, 5, replace=False), rng.choice(np.arange(k, n), m - 5, replace=False)])
        z = mu[idx] + 0.05 * rng.normal(size=(m, q))
    else:
        raise SystemExit(f"unknown case {name}")
    a = rng.normal(size=(m, m))
    adj = (-0.7, rng.normal(size=(m, d)), a + a.T)
    c = z.mean(axis=0)
    tz = float(np.max(np.sum(((z - c) / ls) ** 2, axis=1)))
    t = 1.0 + 2.0 * s / ls**2
    tx = float(np.max(np.sum(((mu - c) / ls) ** 2 / t, axis=1)))
    if not expected:
        t = np.ones_like(s)
        tx = float(np.max(np.sum(((mu - c) / ls) ** 2, axis=1)))
    k = sgp.KernelSpec(1.3, ls)
    ctx = sgp.Context.default()
    ctx.set_precision(os.environ.get("SGPX_PSI_MODE", "auto"))
    st, g = sgp.sweep_stats(expected, mu, s if expected else None, y, z, k, adj=sgp.StatsAdjoints(*adj))
    mode, _ = ctx.last_precision()
    wst, wg = oracle.sweep_stats(expected, mu, s if expected else None, y, z, 1.3, ls, adj=adj)
    pairs = dict(phi=(st.phi_big, wst.phi_big), psi=(st.psi_y, wst.psi_y), dz=(g.d_z, wg.d_z),
                 dl=(g.d_lengthscales, wg.d_lengthscales), dvar=([g.d_variance], [wg.d_variance]))
    if expected:
        pairs.update(dmu=(g.d_mu, wg.d_mu), ds=(g.d_s, wg.d_s))
    el = {k2: rel(*v) for k2, v in pairs.items()}
    nw = {k2: nre(*v) for k2, v in pairs.items()}
    print(f"{name0:18s} {mode:7s} Tz={tz:9.1f} Tx={tx:9.1f} | elem " + " ".join(f"{k2}={v:.1e}" for k2, v in el.items()) +
          " | norm " + " ".join(f"{k2}={v:.1e}" for k2, v in nw.items()), flush=True)


if __name__ == "__main__":
    cases = sys.argv[1:] or ["gauss:1", "gauss:2", "gauss:3", "gauss:4", "gauss:8", "gauss:16", "gauss:24",
                             "gauss:32", "bimodal:10", "bimodal:30", "bimodal:100", "bimodal:300",
                             "farcluster:30", "farcluster:300", "outliers:30", "outliers:300", "outliers:1000",
                             "zcluster:20", "zcluster:60", "det-gauss:1", "det-gauss:2", "det-gauss:4", "det-gauss:8",
                             "det-bimodal:10", "det-bimodal:30", "det-bimodal:300", "det-outliers:1000"]
    print("mode:", os.environ.get("SGPX_PSI_MODE", "auto"))
    for cname in cases:
        try:
            case(cname)
        except Exception as e:  # noqa: BLE001
            print(f"{cname:16s} ERROR {type(e).__name__}: {e}", flush=True)
