"""Row-tile accuracy against the fp64 oracle across latent widths Q, both modes (the parity-test
problem generator: mu ~ N(0, 1), S ~ U(0.25, 1), l ~ U(0.5, 2), Z = M rows of mu + noise)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1410_4984_b200 import sgp  # noqa: E402
from test_gpu_parity import problem, sym_adj  # noqa: E402
from conftest import norm_rel_err as nre  # noqa: E402

oracle.lib()
for n, d, m in ((64, 5, 12), (2000, 6, 50)):
    for q in (8, 10, 12, 16, 18, 20):
        for expected in (True, False):
            mu, s, y, z, var, ls = problem(2, n, q, d, m)
            adj = sym_adj(np.random.default_rng(5), m, d)
            k = sgp.KernelSpec(var, ls)
            st, g = sgp.sweep_stats(expected, mu, s, y, z, k, adj=sgp.StatsAdjoints(*adj))
            wst, wg = oracle.sweep_stats(expected, mu, s if expected else None, y, z, var, ls, adj=adj)
            print(f"n={n} m={m} q={q:2d} exp={int(expected)} phi={nre(st.phi_big, wst.phi_big):.1e} "
                  f"psi={nre(st.psi_y, wst.psi_y):.1e} dz={nre(g.d_z, wg.d_z):.1e} "
                  f"dl={nre(g.d_lengthscales, wg.d_lengthscales):.1e}", flush=True)
