"""Timeline of one end-to-end C3 evaluation (pinned host mu/S in, d_mu/d_S out) from the CUPTI
trace torch.profiler collects: every kernel and memcpy of the process, relative to the first.

  python tools/e2e_timeline.py [--n 1000000]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1410_4984_b200 import sgp, synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--q", type=int, default=10)
ap.add_argument("--d", type=int, default=50)
ap.add_argument("--m", type=int, default=100)
a = ap.parse_args()
dev = torch.device("cuda", 0)
w = synthetic.make(True, a.n, a.q, a.d, a.m, seed=0, device=dev)
mu, s, y, z = w.mu, w.s, w.y, w.z
ctx = sgp.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
eng = sgp.Engine(sgp.ModelKind.latent, mu, s, y, ctx=ctx)
kern = w.kernel
mu_h = torch.empty(a.q, a.n, dtype=torch.float64, pin_memory=True)
s_h = torch.empty(a.q, a.n, dtype=torch.float64, pin_memory=True)
mu_h.copy_(mu.t())
s_h.copy_(s.t())
mu_np, s_np = mu_h.numpy().T, s_h.numpy().T
gmu_h = torch.empty(a.q, a.n, dtype=torch.float64, pin_memory=True)
gs_h = torch.empty(a.q, a.n, dtype=torch.float64, pin_memory=True)
eng.set_local_grads_out(gmu_h.numpy().T, gs_h.numpy().T)
for _ in range(3):
    eng.broadcast(kern, w.beta, z, mu_np, s_np)
    eng.evaluate(True)
torch.cuda.synchronize()
resident = bool(os.environ.get("RESIDENT"))
if resident:  # device-resident rows (the bench's `value` path)
    eng = sgp.Engine(sgp.ModelKind.latent, mu, s, y, ctx=ctx)
    for _ in range(3):
        eng.broadcast(kern, w.beta, z)
        eng.evaluate(True, local_to_host=False)
    torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    if resident:
        eng.broadcast(kern, w.beta, z)
        r = eng.evaluate(True, local_to_host=False)
    else:
        eng.broadcast(kern, w.beta, z, mu_np, s_np)
        r = eng.evaluate(True)
    torch.cuda.synchronize()
events = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in events)
rows = sorted((e.time_range.start - t0, e.time_range.end - t0, e.name) for e in events)
for st, en, name in rows:
    if en - st >= float(os.environ.get("MIN_US", "20")) or "Memcpy" in name:
        print(f"{st / 1e3:8.3f} - {en / 1e3:8.3f} ms  {(en - st) / 1e3:7.3f}  {name[:80]}")
print(f"span {max(r[1] for r in rows) / 1e3:.3f} ms over {len(rows)} device events")
if os.environ.get("CPU_EVENTS"):
    cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cu")]
    c0 = min(e.time_range.start for e in cpu)
    print(f"--- runtime API calls (CPU clock, first at {c0}; device clock first event at {t0})")
    for e in sorted(cpu, key=lambda e: e.time_range.start):
        print(f"{(e.time_range.start - c0) / 1e3:8.3f} ms  {(e.time_range.end - e.time_range.start) / 1e3:7.3f}  {e.name[:60]}")
