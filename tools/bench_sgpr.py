"""Timing of the deterministic (SGPR) evaluation, C4-shaped (BASELINE.json configs[3]: N=10M, Q=8,
D=1, M=500; X, Y ~ N(0,1), Z = M rows of X, sigma^2 = l = beta = 1), device-resident,
CUDA events on the engine's stream.  Not a bench line: BASELINE.json's metric is quoted on C3.
Usage: python tools/bench_sgpr.py [N] [steps]   (SGPX_RT_DET=0 for the direct-difference kernels)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1410_4984_b200 import sgp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
q, d, m = 8, 1, 500
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(q, n, generator=g, device=dev, dtype=torch.float64).t()  # column-major n x q
y = torch.randn(d, n, generator=g, device=dev, dtype=torch.float64).t()
z = x[torch.randperm(n, generator=g, device=dev)[:m]].cpu().numpy()
ctx = sgp.Context(0)
st = torch.cuda.current_stream(dev)
ctx.set_stream(st.cuda_stream)
eng = sgp.Engine(sgp.ModelKind.regression, x, None, y, ctx=ctx)
eng.broadcast(sgp.KernelSpec(1.0, np.ones(q)), 1.0, z)
r = eng.evaluate(True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(steps):
    r = eng.evaluate(True)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
p = m * (m + 1) // 2
print(f"SGPR N={n} Q={q} D={d} M={m}: {ms:.2f} ms/eval, {n / ms * 1e3 / 1e6:.2f} M dp/s, "
      f"bound {r.bound.total:.10e}, fwd {r.timing.fwd_kernel_s * 1e3:.2f} ms, bwd {r.timing.bwd_kernel_s * 1e3:.2f} ms",
      flush=True)
