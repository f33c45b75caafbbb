"""Per-frame wall time and skin-list counters of the value path (state in
HBM) and the e2e path (set_state / run_frames / get_state every frame).

python tools/e2e_probe.py [scene] [settle] [frames]
"""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2605_15875_b200 import _lib as L
    from paper_2605_15875_b200 import api
    from paper_2605_15875_b200.scene import make_scenario

    scene = sys.argv[1] if len(sys.argv) > 1 else "pile-1k"
    settle = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    frames = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    lib = L.load()
    sc = api.Scene(make_scenario(scene))

    def stats(ctx):
        r, n, d = C.c_longlong(), C.c_int(), C.c_double()
        L.check(lib.dabd_gpu_ctx_list_stats(ctx.h, C.byref(r), C.byref(n), C.byref(d)))
        return r.value, n.value, d.value

    ctx = api.Context(sc)
    ctx.run_frames(settle)
    torch.cuda.synchronize()
    q, qd = ctx.state()
    print("value path", stats(ctx))
    for f in range(frames):
        t0 = time.perf_counter()
        st = ctx.run_frames(1)[0]
        dt = time.perf_counter() - t0
        print(f"  frame {f}: {1e3 * dt:7.2f} ms newton {st['newton_iterations']} list {stats(ctx)}")
    ctx2 = api.Context(sc)
    qh = q.copy()
    qdh = qd.copy()
    qp = qh.ctypes.data_as(C.POINTER(C.c_double))
    qdp = qdh.ctypes.data_as(C.POINTER(C.c_double))
    arr = (L.FrameStats * 1)()
    print("e2e path")
    for f in range(frames + 1):
        t0 = time.perf_counter()
        L.check(lib.dabd_gpu_set_state(ctx2.h, qp, qdp))
        t1 = time.perf_counter()
        L.check(lib.dabd_gpu_run_frames(ctx2.h, 1, arr))
        t2 = time.perf_counter()
        L.check(lib.dabd_gpu_get_state(ctx2.h, qp, qdp))
        t3 = time.perf_counter()
        print(f"  frame {f}: set {1e3 * (t1 - t0):6.2f} run {1e3 * (t2 - t1):7.2f} get {1e3 * (t3 - t2):6.2f} ms"
              f" newton {arr[0].newton_iterations} list {stats(ctx2)}")


if __name__ == "__main__":
    main()
