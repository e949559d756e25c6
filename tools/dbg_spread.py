"""Accuracy of the default (row-tile) path against the fp64 oracle as the data spread grows
relative to the lengthscale: mu ~ N(0, f^2), Z = M rows of mu, l ~ U(0.5, 2).  The exponent
features grow like (mu / l)^2, so the 2^-22 piece accuracy turns into an absolute exponent error
that grows with f."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1410_4984_b200 import sgp  # noqa: E402

oracle.lib()


def nre(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


n, q, d, m = 4000, 10, 10, 100
for f in (1.0, 2.0, 4.0, 8.0, 16.0):
    rng = np.random.default_rng(1)
    mu = f * rng.normal(size=(n, q))
    s = rng.uniform(0.25, 1.0, (n, q))
    y = rng.normal(size=(n, d))
    z = mu[rng.choice(n, m, replace=False)] + 0.05 * rng.normal(size=(m, q))
    ls = rng.uniform(0.5, 2.0, q)
    a = rng.normal(size=(m, m))
    adj = (-0.7, rng.normal(size=(m, d)), a + a.T)
    k = sgp.KernelSpec(1.3, ls)
    st, g = sgp.sweep_stats(True, mu, s, y, z, k, adj=sgp.StatsAdjoints(*adj))
    wst, wg = oracle.sweep_stats(True, mu, s, y, z, 1.3, ls, adj=adj)
    out = dict(phi_big=nre(st.phi_big, wst.phi_big), psi_y=nre(st.psi_y, wst.psi_y), dz=nre(g.d_z, wg.d_z),
               dl=nre(g.d_lengthscales, wg.d_lengthscales), dvar=nre(g.d_variance, wg.d_variance),
               dmu=nre(g.d_mu, wg.d_mu), ds=nre(g.d_s, wg.d_s))
    print(f"spread {f:5.1f}", " ".join(f"{kk}={v:.1e}" for kk, v in out.items()), flush=True)
