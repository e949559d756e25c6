"""A few C3 evaluations (device-resident Rng inputs) for launch lists under ncu / timelines.
Usage: python tools/one_eval.py [evals] [N Q D M]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1410_4984_b200 import sgp, synthetic  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n, q, d, m = (int(x) for x in (sys.argv[2:6] if len(sys.argv) >= 6 else (1_000_000, 10, 50, 100)))
w = synthetic.make(True, n, q, d, m, seed=0, device="cuda")
eng = sgp.Engine(sgp.ModelKind.latent, w.mu, w.s, w.y, precision=os.environ.get("PREC", "auto"))
eng.broadcast(w.kernel, w.beta, w.z)
for _ in range(k):
    r = eng.evaluate(True, local_to_host=False)
torch.cuda.synchronize()
t = r.timing
print(f"coordinator {t.coordinator_s * 1e3:.3f} ms  fwd {t.fwd_kernel_s * 1e3:.3f}  bwd {t.bwd_kernel_s * 1e3:.3f}  "
      f"stats pass {t.stats_pass_s * 1e3:.3f}  grad pass {t.grad_pass_s * 1e3:.3f}  wall {t.wall_s * 1e3:.3f}")
