import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tests"))
import numpy as np
import oracle as orc
from paper_1410_4984_b200 import sgp, synthetic
from conftest import rel_err
for shape in [(20_011, 6, 17, 40), (50_000, 10, 50, 100)]:
    n, q, d, m = shape
    w = synthetic.make(True, n, q, d, m, seed=31)
    ref = orc.engine_evaluate(True, w.mu, w.s, w.y, w.z, w.variance, w.lengthscales, w.beta, workers=os.cpu_count())
    for old in ("0", "1"):
        if old == "1": os.environ["SGPX_PSI1_BWD"] = "old"
        else: os.environ.pop("SGPX_PSI1_BWD", None)
        eng = sgp.Engine(sgp.ModelKind.latent, w.mu, w.s, w.y)
        eng.broadcast(w.kernel, w.beta, w.z)
        r = eng.evaluate(True)
        dz = r.grads.d_z; rz = ref.d_z
        e = np.abs(dz - rz) / np.maximum(np.abs(rz), 1e-300)
        i = np.unravel_index(np.argmax(e), e.shape)
        print(shape, "old" if old == "1" else "pipe", "dz max elem rel", e.max(), "at", i, dz[i], rz[i], "max|dz|", np.abs(rz).max(), "prec", r.precision_used if hasattr(r, "precision_used") else "")
        eng.close()
