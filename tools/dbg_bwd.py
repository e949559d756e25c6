import sys, os, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from test_gpu_parity import problem, sym_adj
import oracle
from paper_1410_4984_b200 import sgp
for shape in [(300, 3, 4, 7), (257, 10, 10, 100), (64, 20, 5, 12), (33, 2, 1, 5)]:
    n, q, d, m = shape
    mu, s, y, z, var, ls = problem(2, n, q, d, m)
    adj = sym_adj(np.random.default_rng(5), m, d)
    st, g = sgp.sweep_stats(True, mu, s, y, z, sgp.KernelSpec(var, ls), adj=sgp.StatsAdjoints(*adj))
    wst, wg = oracle.sweep_stats(True, mu, s, y, z, var, ls, adj=adj)
    nr = lambda a, b: float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))
    print(shape, 'dvar', g.d_variance, wg.d_variance, 'dz', nr(g.d_z, wg.d_z), 'dl', nr(g.d_lengthscales, wg.d_lengthscales),
          'dmu', nr(g.d_mu, wg.d_mu), 'ds', nr(g.d_s, wg.d_s))
