"""Criterion-3 sweep (every builtin x N frames) that reports the first
failing scene/frame and its error instead of stopping at an assertion."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    from paper_2605_15875_b200 import api
    from paper_2605_15875_b200.scene import make_scenario
    from test_gpu_acceptance import BUILTINS

    frames = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    names = sys.argv[2:] or BUILTINS
    for name in names:
        sd = make_scenario(name)
        workers = {"drop-grid-1": 1, "drop-grid-4": 4}.get(name, 2)
        ctx = api.Context(api.Scene(sd), num_workers=workers)
        t = time.time()
        for f in range(frames):
            try:
                st = ctx.run_frames(1)[0]
                if os.environ.get("CRIT3_AUDIT", "1") == "1":
                    hit, nviol, _ = ctx.audit()
                    if hit or nviol:
                        print(name, "frame", f, "audit: intersecting", hit, "violating", nviol, flush=True)
            except Exception as e:  # noqa: BLE001
                print(name, "frame", f, "error:", e, flush=True)
                if "illegal" in str(e) or "CUDA error" in str(e):
                    return
                break
        else:
            print(name, "ok", frames, f"{time.time() - t:.1f}s", flush=True)


if __name__ == "__main__":
    main()
