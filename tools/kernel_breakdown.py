"""Per-kernel time breakdown of the hot path (CUDA events around every
dabd_gpu launch, eager mode) next to the graph-mode step time.

python tools/kernel_breakdown.py [scene] [settle] [frames]
"""

import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    scene = sys.argv[1] if len(sys.argv) > 1 else "pile-1k"
    settle = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    frames = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    from paper_2605_15875_b200 import _lib as L
    from paper_2605_15875_b200 import api
    from paper_2605_15875_b200.scene import make_scenario

    lib = L.load()
    sd = make_scenario(scene)
    sc = api.Scene(sd)
    out = {"scene": scene, "settle": settle, "frames": frames}
    for mode in ("graph", "eager"):
        os.environ["DABD_GPU_NO_GRAPH"] = "1" if mode == "eager" else "0"
        ctx = api.Context(sc)
        ctx.run_frames(settle)
        torch.cuda.synchronize()
        if mode == "eager":
            lib.dabd_gpu_kernel_timer_enable(b"*")
        t0 = time.perf_counter()
        st = ctx.run_frames(frames)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / frames
        out[mode] = {"ms_per_frame_wall": 1e3 * dt, "stats": st}
        if mode == "eager":
            buf = C.create_string_buffer(1 << 16)
            lib.dabd_gpu_kernel_timer_report(buf, 1 << 16)
            lib.dabd_gpu_kernel_timer_enable(None)
            rows = []
            for item in buf.value.decode().split(";"):
                if item.strip():
                    n, c, ms = item.split()
                    rows.append((n, int(c), float(ms)))
            tot = sum(r[2] for r in rows)
            rows.sort(key=lambda r: -r[2])
            out["eager"]["kernels"] = [
                {"kernel": n, "launches_per_frame": c / frames, "ms_per_frame": ms / frames,
                 "share": ms / tot, "avg_us": 1e3 * ms / max(c, 1)} for n, c, ms in rows]
            out["eager"]["kernel_ms_per_frame"] = tot / frames
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
