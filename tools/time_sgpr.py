"""SGPR (deterministic inputs) evaluation time per mode at the C4 shape: Q=8, D=1, M=500.
Usage: python tools/time_sgpr.py [N]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1410_4984_b200 import sgp, synthetic  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
w = synthetic.make(False, n, 8, 1, 500, seed=0, device="cuda")
for mode in sys.argv[2:] or ("syrk", "precise"):
    eng = sgp.Engine(sgp.ModelKind.regression, w.mu, None, w.y, precision=mode)
    eng.broadcast(w.kernel, w.beta, w.z)
    r = eng.evaluate(True, local_to_host=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    k = 3
    for _ in range(k):
        r = eng.evaluate(True, local_to_host=False)
    dt = (time.perf_counter() - t0) / k
    t = r.timing
    print(f"N={n} {mode:8s} used={t.precision:8s} {dt * 1e3:9.2f} ms/eval  fwd {t.fwd_kernel_s * 1e3:8.2f}  "
          f"bwd {t.bwd_kernel_s * 1e3:8.2f}  stats {t.stats_pass_s * 1e3:8.2f}  coord {t.coordinator_s * 1e3:8.2f}  "
          f"grad {t.grad_pass_s * 1e3:8.2f}  bound {r.bound.total:.12e}  {n / dt / 1e6:.2f} M dp/s", flush=True)
    eng.close()
