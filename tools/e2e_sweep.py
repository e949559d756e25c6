"""End-to-end C3 evaluation time (pinned host mu/S uploaded by broadcast(), d_mu/d_S streamed back)
for a list of sub-shard plans (SGPX_SUBS) and coordinator placements (SGPX_DEVICE_COORD).

  [E2E_SHAPE=n,q,d,m] python tools/e2e_sweep.py [steps] "plan1" "plan2" ...
  plan = "<subs>|<devcoord 0/1>[|NAME=v,...]", e.g. "1,2,2|0"
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1410_4984_b200 import sgp, synthetic  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
plans = sys.argv[2:] or ["|0", "|1"]
n, q, d, m = (int(x) for x in os.environ.get("E2E_SHAPE", "1000000,10,50,100").split(","))  # C3 by default
w = synthetic.make(True, n, q, d, m, seed=0, device="cuda")
mu_p = torch.empty(q, n, dtype=torch.float64, pin_memory=True)
s_p = torch.empty(q, n, dtype=torch.float64, pin_memory=True)
mu_p.copy_(w.mu.t())
s_p.copy_(w.s.t())
mu_np, s_np = mu_p.numpy().T, s_p.numpy().T
gmu_p = torch.empty(q, n, dtype=torch.float64, pin_memory=True)
gs_p = torch.empty(q, n, dtype=torch.float64, pin_memory=True)
for plan in plans:
    subs, _, rest = plan.partition("|")
    dc, _, extra = rest.partition("|")  # optional third field: NAME=value set for this plan
    for kv in filter(None, extra.split(",")):
        name, _, val = kv.partition("=")
        os.environ[name] = val
    if subs:
        os.environ["SGPX_SUBS"] = subs
    else:
        os.environ.pop("SGPX_SUBS", None)
    if dc:
        os.environ["SGPX_DEVICE_COORD"] = dc
    else:
        os.environ.pop("SGPX_DEVICE_COORD", None)
    ctx = sgp.Context(0)  # an explicit stream, as bench.py (the graph-replayed path)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    eng = sgp.Engine(sgp.ModelKind.latent, w.mu, w.s, w.y, ctx=ctx)
    eng.set_local_grads_out(gmu_p.numpy().T, gs_p.numpy().T)
    ts, tb = [], []
    for i in range(steps + 2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.broadcast(w.kernel, w.beta, w.z, mu_np, s_np)
        t1 = time.perf_counter()
        r = eng.evaluate(True)
        _ = r.bound.total
        ts.append(time.perf_counter() - t0)
        tb.append(t1 - t0)
    ts, tb = sorted(ts[2:]), sorted(tb[2:])
    print(f"plan {plan:28s} e2e median {ts[len(ts) // 2] * 1e3:7.3f} ms  min {ts[0] * 1e3:7.3f}  "
          f"(broadcast {tb[len(tb) // 2] * 1e3:6.3f} ms)  bound {r.bound.total:.10e}", flush=True)
    del eng
