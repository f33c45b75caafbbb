"""Frames/s and solver counts of the larger BASELINE.json configs on ONE GPU
(partitions batched on the device), plus the device audit of the final
state (intersection_test + minimum point-edge distance, dabd_gpu_audit).

python tools/scale_probe.py scene:workers:frames [...]
   e.g. pour-10k:8:20 sweep-100k:8:5 hetero-1000:2:20 cubes-64:2:50
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2605_15875_b200 import api
    from paper_2605_15875_b200.scene import make_scenario

    for spec in sys.argv[1:]:
        name, workers, frames = spec.split(":")
        workers, frames = int(workers), int(frames)
        sd = make_scenario(name)
        t0 = time.perf_counter()
        sc = api.Scene(sd)
        ctx = api.Context(sc, num_workers=workers)
        ctx.run_frames(1)  # capture / first-touch outside the timing
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        st = ctx.run_frames(frames)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t1
        t2 = time.perf_counter()
        hit, nviol, dmin = ctx.audit(None, cutoff=sd.params.d_hat)  # device state, no copies
        t_audit = time.perf_counter() - t2
        out = {
            "scene": name, "bodies": sc.n, "workers": workers, "frames": frames,
            "setup_s": t1 - t0, "ms_per_frame": 1e3 * dt / frames, "steps_per_s": frames / dt,
            "admm_per_frame": sum(s["admm_iterations"] for s in st) / frames,
            "newton_per_frame": sum(s["newton_iterations"] for s in st) / frames,
            "pcg_per_frame": sum(s["pcg_iterations"] for s in st) / frames,
            "attempts": sum(s["attempts"] for s in st), "committed": sum(s["committed"] for s in st),
            "max_contacts": max(s["max_contacts"] for s in st),
            "intersecting_end": hit, "violating_pairs_end": nviol, "min_distance_end": dmin,
            "audit_ms": 1e3 * t_audit,
            # per-frame wall split (FrameStats): the solve graph vs host setup + commit
            "t_frame_ms": 1e3 * sum(s["t_frame"] for s in st) / frames,
            "t_solve_ms": 1e3 * sum(s["t_solve"] for s in st) / frames,
            "host_setup_frac": 1.0 - sum(s["t_solve"] for s in st) / max(sum(s["t_frame"] for s in st), 1e-12),
        }
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
