"""Per-block parity of Engine::evaluate(true) in each precision mode at the benchmark shapes
(Rng inputs): element-wise rel_err (oracles.hpp:55-58) with the worst element, its magnitude and the
block's max magnitude, and the norm-wise error.  Usage: python tools/dbg_parity_modes.py C2|C4|C3 [N]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1410_4984_b200 import sgp, synthetic  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
shapes = {"C2": (True, 100_000, 10, 10, 100), "C3": (True, 1_000_000, 10, 50, 100), "C4": (False, 20_000, 8, 1, 500),
          "C5": (True, 20_000, 20, 100, 256)}
latent, n, q, d, m = shapes[cfg]
if len(sys.argv) > 2:
    n = int(sys.argv[2])
w = synthetic.make(latent, n, q, d, m, seed=0)
ref = oracle.engine_evaluate(latent, w.mu, w.s, w.y, w.z, w.variance, w.lengthscales, w.beta, workers=os.cpu_count())
for mode in ("fast", "precise", "direct"):
    e = sgp.Engine(sgp.ModelKind.latent if latent else sgp.ModelKind.regression, w.mu, w.s, w.y, precision=mode)
    e.broadcast(w.kernel, w.beta, w.z)
    r = e.evaluate(True)
    out = [f"{cfg} N={n} {mode:8s}({r.timing.precision}) bound {abs(r.bound.total - ref.bound['total']) / abs(ref.bound['total']):.1e}"]
    blocks = dict(d_z=(r.grads.d_z, ref.d_z), d_ls=(r.grads.d_lengthscales, ref.d_lengthscales))
    if latent:
        blocks.update(d_mu=(r.grads.d_mu, ref.d_mu), d_s=(r.grads.d_s, ref.d_s))
    for k, (a, b) in blocks.items():
        a, b = np.ravel(a), np.ravel(b)
        el = np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)
        i = int(np.argmax(el))
        out.append(f"{k}: elem {el[i]:.1e} at |{b[i]:.2e}| (max {np.max(np.abs(b)):.2e}) norm "
                   f"{np.linalg.norm(a - b) / np.linalg.norm(b):.1e}")
    print(" | ".join(out), flush=True)
    e.close()
