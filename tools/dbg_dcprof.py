import ctypes as C, sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_1410_4984_b200 import sgp, synthetic, _lib
w = synthetic.make(True, 100000, 10, 50, 100, seed=0, device="cuda")
os.environ["SGPX_GRAPH"] = "0"
os.environ.setdefault("SGPX_DEVICE_COORD", "1")
e = sgp.Engine(sgp.ModelKind.latent, w.mu, w.s, w.y)
e.broadcast(w.kernel, w.beta, w.z)
for _ in range(3):
    r = e.evaluate(True, local_to_host=False)
a = (C.c_longlong * 16)()
_lib.load().sgpx_debug_dc_profile(a)
print("phase cycles:", [a[i + 1] - a[i] for i in range(5)], "panel0:", [a[5] - a[1], a[6] - a[5], a[7] - a[6], a[8] - a[7]], "attempts", a[10], a[11], "ok", a[12], a[13], "coord", r.timing.coordinator_s)
