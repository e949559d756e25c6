"""Direct mode through the engine: device-resident (one sub-shard) vs host buffers (sub-shards)
vs the one-shot sweep, against the oracle, on the bimodal +-300 l latent space."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1410_4984_b200 import sgp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 520_000
q, d, m = 3, 2, 12
rng = np.random.default_rng(3)
mu = rng.normal(size=(n, q))
mu[:, 0] += np.where(np.arange(n) % 2 == 0, 300.0, -300.0)
s = rng.uniform(0.25, 1.0, (n, q))
y = rng.normal(size=(n, d))
z = mu[rng.choice(n, m, replace=False)]
ls = np.ones(q)
k = sgp.KernelSpec(1.0, ls)
ref = oracle.engine_evaluate(True, mu, s, y, z, 1.0, ls, 20.0, workers=os.cpu_count())
print("oracle d_z[:, 0]", ref.d_z[:, 0])
# host-buffer engine (sub-shards when n >= 500k)
e = sgp.Engine(sgp.ModelKind.latent, mu, s, y)
e.broadcast(k, 20.0, z, mu, s)
r = e.evaluate(True)
print("host   ", r.timing.precision, "d_z[:, 0]", r.grads.d_z[:, 0])
# device-resident engine
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()  # noqa: E731
mt, st_, yt = dev(mu), dev(s), dev(y)
e2 = sgp.Engine(sgp.ModelKind.latent, mt, st_, yt)
e2.broadcast(k, 20.0, z)
r2 = e2.evaluate(True)
print("device ", r2.timing.precision, "d_z[:, 0]", r2.grads.d_z[:, 0])
for name, rr in (("host", r), ("device", r2)):
    for f in ("d_z", "d_mu", "d_s", "d_lengthscales"):
        a, b = np.asarray(getattr(rr.grads, f)), np.asarray(getattr(ref, f))
        print(name, f, float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0))))
    print(name, "bound", rr.bound.total, ref.bound["total"])
