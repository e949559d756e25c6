"""Row-tile psi2 path vs the oracle: per-output errors on a few shapes (GPU)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1410_4984_b200 import sgp  # noqa: E402

oracle.lib()


def nre(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


shapes = [(300, 3, 4, 7), (1, 1, 1, 1), (257, 10, 10, 100), (1000, 8, 2, 33), (64, 20, 5, 12), (5000, 10, 10, 100)]
for expected in (True, False):
    for (n, q, d, m) in shapes:
        rng = np.random.default_rng(1)
        mu = rng.normal(size=(n, q))
        s = rng.uniform(0.25, 1.0, (n, q))
        y = rng.normal(size=(n, d))
        z = mu[rng.choice(n, m, replace=n < m)] + 0.05 * rng.normal(size=(m, q))
        ls = rng.uniform(0.5, 2.0, q)
        a = rng.normal(size=(m, m))
        adj = (-0.7, rng.normal(size=(m, d)), a + a.T)
        k = sgp.KernelSpec(1.3, ls)
        st, g = sgp.sweep_stats(expected, mu, s, y, z, k, adj=sgp.StatsAdjoints(*adj))
        wst, wg = oracle.sweep_stats(expected, mu, s if expected else None, y, z, 1.3, ls, adj=adj)
        out = dict(phi_big=nre(st.phi_big, wst.phi_big), psi_y=nre(st.psi_y, wst.psi_y) if d else 0,
                   dz=nre(g.d_z, wg.d_z), dl=nre(g.d_lengthscales, wg.d_lengthscales),
                   dvar=nre(g.d_variance, wg.d_variance))
        if expected:
            out.update(dmu=nre(g.d_mu, wg.d_mu), ds=nre(g.d_s, wg.d_s))
        print(("E" if expected else "D"), (n, q, d, m), " ".join(f"{k}={v:.1e}" for k, v in out.items()), flush=True)
