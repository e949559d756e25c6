"""Host vs device coordinator vs oracle at a large-M SGPR shape (debug).
Usage: python tools/dbg_coord_large_m.py [q] [m] [precision]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1410_4984_b200 import sgp, synthetic  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


q = int(sys.argv[1]) if len(sys.argv) > 1 else 4
m = int(sys.argv[2]) if len(sys.argv) > 2 else 500
prec = sys.argv[3] if len(sys.argv) > 3 else "direct"
w = synthetic.make(False, 30_000, q, 8, m, seed=4)
out = {}
for dev in ("1", "0"):
    os.environ["SGPX_DEVICE_COORD"] = dev
    eng = sgp.Engine(sgp.ModelKind.regression, w.mu, w.s, w.y, precision=prec)
    eng.broadcast(w.kernel, w.beta, w.z)
    out[dev] = eng.evaluate(True)
    eng.close()
ref = oracle.engine_evaluate(False, w.mu, None, w.y, w.z, w.variance, w.lengthscales, w.beta,
                             workers=os.cpu_count() or 1)
for k, r in out.items():
    print(f"device_coord={k} jitter={r.jitter_factor}  bound {rel(r.bound.total, ref.bound['total']):.3e}  "
          f"dz {rel(r.grads.d_z, ref.d_z):.3e}  dl {rel(r.grads.d_lengthscales, ref.d_lengthscales):.3e}  "
          f"dvar {rel(r.grads.d_variance, ref.d_variance):.3e}  dbeta {rel(r.grads.d_beta, ref.d_beta):.3e}")
print("dev vs host dz", rel(out["1"].grads.d_z, out["0"].grads.d_z))
