"""Device-resident C3-shaped evaluation time at a shard size (the per-GPU work of an N-GPU strong-
scaling run: N = 1M / GPUs), CUDA events on the engine's stream.  Compare the coordinators with
SGPX_DEVICE_COORD=0|1.
Usage: python tools/time_shard.py [n ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1410_4984_b200 import sgp, synthetic  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [1_000_000, 500_000, 250_000, 125_000]:
    w = synthetic.make(True, n, 10, 50, 100, seed=0, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        ctx = sgp.Context(0)
        ctx.set_stream(st.cuda_stream)
        eng = sgp.Engine(sgp.ModelKind.latent, w.mu, w.s, w.y, ctx=ctx)
        eng.broadcast(w.kernel, w.beta, w.z)
        for _ in range(3):
            r = eng.evaluate(True, local_to_host=False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k = 20
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(k):
            r = eng.evaluate(True, local_to_host=False)
        e1.record(st)
        torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / k
    print(f"N={n:8d}  {t:7.3f} ms/eval  kernels fwd {r.timing.fwd_kernel_s * 1e3:6.3f} bwd {r.timing.bwd_kernel_s * 1e3:6.3f}"
          f"  coord {r.timing.coordinator_s * 1e3:6.3f} ms  device_coord={os.environ.get('SGPX_DEVICE_COORD', 'default')}",
          flush=True)
    eng.close()
