"""Evaluation time of each precision mode at a benchmark shape (device-resident inputs, CUDA-event
timed passes).  Usage: python tools/time_modes.py [N Q D M]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1410_4984_b200 import sgp, synthetic  # noqa: E402

n, q, d, m = (int(x) for x in (sys.argv[1:5] if len(sys.argv) >= 5 else (1_000_000, 10, 50, 100)))
latent = os.environ.get("KIND", "latent") == "latent"
w = synthetic.make(latent, n, q, d, m, seed=0, device="cuda")
for mode in ("fast", "precise", "direct"):
    eng = sgp.Engine(sgp.ModelKind.latent if latent else sgp.ModelKind.regression, w.mu, w.s, w.y,
                     precision=mode)
    eng.broadcast(w.kernel, w.beta, w.z)
    for _ in range(2):
        r = eng.evaluate(True, local_to_host=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    k = 3
    for _ in range(k):
        r = eng.evaluate(True, local_to_host=False)
    dt = (time.perf_counter() - t0) / k
    t = r.timing
    print(f"{mode:8s} used={t.precision:8s} wall {dt*1e3:8.2f} ms  fwd {t.fwd_kernel_s*1e3:7.2f} ms  "
          f"bwd {t.bwd_kernel_s*1e3:7.2f} ms  bound {r.bound.total:.10e}  {n / dt / 1e6:.2f} M dp/s", flush=True)
    eng.close()
