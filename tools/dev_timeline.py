import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from torch.profiler import ProfilerActivity, profile
from paper_1410_4984_b200 import sgp, synthetic
w = synthetic.make(True, 1_000_000, 10, 50, 100, seed=0, device="cuda")
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    ctx = sgp.Context(0); ctx.set_stream(st.cuda_stream)
    eng = sgp.Engine(sgp.ModelKind.latent, w.mu, w.s, w.y, ctx=ctx)
    eng.broadcast(w.kernel, w.beta, w.z)
    for _ in range(3): eng.evaluate(True, local_to_host=False)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        eng.evaluate(True, local_to_host=False)
        torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in ev)
rows = sorted((e.time_range.start - t0, e.time_range.end - t0, e.name) for e in ev)
prev = 0
for a, b, n in rows:
    print(f"{a/1e3:7.3f}-{b/1e3:7.3f} {(b-a)/1e3:6.3f} gap {(a-prev)/1e3:6.3f} {n[:70]}")
    prev = b
