"""Row-tile kernel timing experiments (SGPX_RT_DBG: 1 skip the consumers' G math, 2 skip MMA3, 4 skip
MMA1, 8 TMEM traffic without exp2): one sweep_stats forward + backward at the C3 shape; run under
`ncu --metrics gpu__time_duration.sum` to read the kernel times (the results are garbage by design).
Usage: SGPX_RT_DBG=k python tools/rt_dbg_time.py [n]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1410_4984_b200 import sgp, synthetic  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
w = synthetic.make(True, n, 10, 50, 100, seed=0)
rng = np.random.default_rng(1)
a = rng.normal(size=(100, 100)) * 1e-3
adj = sgp.StatsAdjoints(-0.5, rng.normal(size=(100, 50)) * 1e-3, a + a.T)
for _ in range(2):
    sgp.sweep_stats(True, w.mu, w.s, w.y, w.z, w.kernel, adj=adj)
print("done")
