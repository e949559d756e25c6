"""One C3 bound+gradient evaluation on cuda:0 (device-resident inputs), for ncu captures.

  python tools/profile_step.py [--n 1000000] [--evals 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1410_4984_b200 import sgp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--q", type=int, default=10)
ap.add_argument("--d", type=int, default=50)
ap.add_argument("--m", type=int, default=100)
ap.add_argument("--evals", type=int, default=2)
a = ap.parse_args()
dev = torch.device("cuda", 0)
mu, s, y, z = bench.synth_shard(a.n, a.q, a.d, a.m, 0, a.n, dev)
ctx = sgp.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
eng = sgp.Engine(sgp.ModelKind.latent, mu, s, y, ctx=ctx)
eng.broadcast(sgp.KernelSpec(1.0, np.ones(a.q)), 100.0, z)
for i in range(a.evals):
    r = eng.evaluate(True, local_to_host=False)
torch.cuda.synchronize()
print(f"bound {r.bound.total:.6e} fwd {r.timing.fwd_kernel_s*1e3:.3f} ms bwd {r.timing.bwd_kernel_s*1e3:.3f} ms "
      f"grids {r.timing.fwd_grid}/{r.timing.bwd_grid}")
