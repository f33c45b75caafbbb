"""Device-side vs host-driven multi-partition ADMM frames (DABD_GPU_ADMM_HOST):
ms per frame, ADMM/Newton counts and the largest state difference between the
two paths, on a settled scene.

python tools/admm_ab.py scene workers settle frames
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2605_15875_b200 import api
    from paper_2605_15875_b200.scene import make_scenario

    name = sys.argv[1] if len(sys.argv) > 1 else "pour-10k"
    workers = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    settle = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    frames = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    sd = make_scenario(name)
    sc = api.Scene(sd)
    ctx = api.Context(sc)
    if settle:
        ctx.run_frames(settle)
    q0, qd0 = ctx.state()
    res = {}
    for mode in ("1", "0"):  # host loop first, then the device loop
        os.environ["DABD_GPU_ADMM_HOST"] = mode
        c = api.Context(sc, num_workers=workers)
        c.set_state(q0, qd0)
        c.run_frames(1)  # first touch / capture
        torch.cuda.synchronize()
        t = time.perf_counter()
        st = c.run_frames(frames)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        q, _ = c.state()
        res[mode] = (q, st, dt, c.take_trace())
        print(json.dumps({"scene": name, "workers": workers, "loop": "host" if mode == "1" else "device",
                          "ms_per_frame": 1e3 * dt / frames,
                          "admm": [s["admm_iterations"] for s in st],
                          "newton": [s["newton_iterations"] for s in st],
                          "attempts": [s["attempts"] for s in st]}), flush=True)
    dq = float(np.abs(res["1"][0] - res["0"][0]).max())
    tr_h, tr_d = res["1"][3], res["0"][3]
    same_trace = tr_h.shape == tr_d.shape and bool(np.array_equal(tr_h, tr_d))
    print(json.dumps({"max_state_diff": dq, "bitwise_state": dq == 0.0, "trace_identical": same_trace,
                      "speedup": res["1"][2] / res["0"][2]}), flush=True)
    os.environ.pop("DABD_GPU_ADMM_HOST", None)


if __name__ == "__main__":
    main()
