"""Cycles per PCG iteration by phase (CTA 0 / warp 0 of the cluster kernel),
from dabd_gpu_ctx_pcg_phases, over a few settled pile frames."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2605_15875_b200 import _lib as L
    from paper_2605_15875_b200 import api
    from paper_2605_15875_b200.scene import make_scenario

    lib = L.load()
    scene = sys.argv[1] if len(sys.argv) > 1 else "pile-1k"
    specs = sys.argv[2:] or ["0:0"]
    for spec in specs:
        os.environ["DABD_GPU_PCG_PHASES"] = "1:" + spec  # read at context creation
        print(f"== timed thread: CTA:warp {spec}")
        one(lib, L, api, make_scenario, scene, torch)


def one(lib, L, api, make_scenario, scene, torch):
    sd = make_scenario(scene)
    ctx = api.Context(api.Scene(sd))
    if scene == "pile-1k":
        from bench import start_state
        ctx.set_state(*start_state(sd, 1))
        ctx.run_frames(3)
    else:
        ctx.run_frames(40)
    torch.cuda.synchronize()
    cyc = (C.c_double * 24)()
    L.check(lib.dabd_gpu_ctx_pcg_phases(ctx.h, 1, cyc))
    ctx.run_frames(4)
    torch.cuda.synchronize()
    ns, n, b, its = C.c_double(), C.c_longlong(), C.c_double(), C.c_longlong()
    L.check(lib.dabd_gpu_ctx_pcg_perf(ctx.h, 0, C.byref(ns), C.byref(n), C.byref(b), C.byref(its)))
    L.check(lib.dabd_gpu_ctx_pcg_phases(ctx.h, 1, cyc))
    it = cyc[7]
    names = ["m=Dinv w + partials", "CTA reduce + push", "arrive", "local SpMV", "wait", "fold+scalars",
             "remote SpMV + recurrences", "iterations"]
    tot = sum(cyc[k] for k in range(7))
    print(f"iterations {it:.0f}, cycles/iteration {tot / max(it, 1):.0f}")
    for k in range(7):
        print(f"  [{k}] {names[k]:28s} {cyc[k] / max(it, 1):8.0f} cyc/it  {100 * cyc[k] / max(tot, 1):5.1f}%")
    nl = max(n.value, 1)
    print(f"launches {n.value}, avg launch {ns.value / nl / 1e3:.1f} us; per launch: setup "
          f"{cyc[8] / nl:.0f} cycles, epilogue {cyc[9] / nl:.0f} cycles")
    sub = ["params (ps, row offsets)", "block counts", "staging issue", "first cluster barrier",
           "exchange plan .. plan barrier", "eps, factor, init"]
    for k in range(6):
        print(f"    setup[{k}] {sub[k]:24s} {cyc[10 + k] / nl:8.0f} cycles/launch")
    for k, nm in enumerate(["eps + send plan", "warm start", "u = Dinv r + barrier", "initial SpMV + m"]):
        print(f"      init[{k}] {nm:22s} {cyc[16 + k] / nl:8.0f} cycles/launch")


if __name__ == "__main__":
    main()
