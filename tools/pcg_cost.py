"""Fixed vs per-iteration cost of the cluster PCG launch: settle pile-1k, then
run frames with the PCG capped at K iterations and read the device-side launch
accounting (dabd_gpu_ctx_pcg_perf)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_15875_b200 import _lib as L
from paper_2605_15875_b200 import api
from paper_2605_15875_b200.scene import make_scenario

lib = L.load()
sd = make_scenario(sys.argv[1] if len(sys.argv) > 1 else "pile-1k")
ctx = api.Context(api.Scene(sd), device=0, num_workers=0)
ctx.run_frames(40)
q, qd = ctx.state()


def perf(reset):
    ns, n, b, it = C.c_double(), C.c_longlong(), C.c_double(), C.c_longlong()
    L.check(lib.dabd_gpu_ctx_pcg_perf(ctx.h, int(reset), C.byref(ns), C.byref(n), C.byref(b), C.byref(it)))
    return ns.value, n.value, b.value, it.value


for k in (1, 2, 5, 10, 20, 40, 80):
    ctx.set_solver(1e-30, k)
    ctx.set_state(q, qd)
    perf(True)
    try:
        ctx.run_frames(1)
    except Exception as e:  # capped PCG may break the Newton line search
        print("k", k, "frame failed:", str(e)[:80])
    ns, n, b, it = perf(True)
    if n:
        print(f"max_iters {k:3d}: launches {n:4d} avg {ns / n / 1e3:8.2f} us  iters/launch {it / n:6.1f}  "
              f"us/iter {ns / max(it, 1) / 1e3:6.2f}", flush=True)

# per-phase cycles of CTA 0 / warp 0 (dabd_gpu_ctx_pcg_phases)
ctx.set_solver(1e-10, 4000)
ctx.set_state(q, qd)
perf(True)
ctx.run_frames(2)
ph = (C.c_double * 8)()
L.check(lib.dabd_gpu_ctx_pcg_phases(ctx.h, 1, ph))
names = ["local m,partials", "cta reduce+push", "arrive", "local spmv", "wait", "fold+scalars",
         "remote spmv+update", "(loop top)"]
iters = max(ph[7], 1)
print(f"phases over {int(ph[7])} iterations (cycles/iteration):")
for k in range(7):
    print(f"  {names[k]:22s} {ph[k] / iters:8.1f}")
