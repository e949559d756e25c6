import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
from paper_1410_4984_b200 import sgp, synthetic
n, q, d, m = (int(x) for x in sys.argv[1:5])
w = synthetic.make(True, n, q, d, m, seed=41, device="cuda")
for env in ["", "SGPX_PHASED=0", "SGPX_COORD_SPLIT=0"]:
    for k in ("SGPX_PSI1_BWD", "SGPX_DEVICE_COORD", "SGPX_COORD_SPLIT", "SGPX_PSI1", "SGPX_RT_PREP", "SGPX_KP", "SGPX_PHASED"):
        os.environ.pop(k, None)
    if env:
        a, b = env.split("=")
        os.environ[a] = b
    e = sgp.Engine(sgp.ModelKind.latent, w.mu, w.s, w.y)
    e.broadcast(w.kernel, w.beta, w.z)
    r = e.evaluate(True)
    dm = r.grads.d_mu
    bad = np.argwhere(~np.isfinite(dm))
    print(f"{env or 'default':24s} bound {r.bound.total:.6e} dmu nan rows {len(np.unique(bad[:, 0])) if len(bad) else 0} first {bad[:1].tolist()} dl {np.isfinite(r.grads.d_lengthscales).all()} prec {r.precision_used if hasattr(r, 'precision_used') else ''}", flush=True)
    e.close()
