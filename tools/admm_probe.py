"""Time consensus-ADMM frames of a scene with W partitions batched on one GPU."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_15875_b200 import api
from paper_2605_15875_b200.scene import make_scenario

ap = argparse.ArgumentParser()
ap.add_argument("--scene", default="pour-10k")
ap.add_argument("--workers", type=int, default=8)
ap.add_argument("--frames", type=int, default=10)
ap.add_argument("--settle", type=int, default=0)
a = ap.parse_args()
sd = make_scenario(a.scene)
ctx = api.Context(api.Scene(sd), device=0, num_workers=a.workers)
if a.settle:
    t0 = time.perf_counter()
    ctx.run_frames(a.settle)
    print(f"settle {a.settle} frames {time.perf_counter() - t0:.2f}s", flush=True)
for f in range(a.frames):
    t0 = time.perf_counter()
    st = ctx.run_frames(1)[0]
    dt = time.perf_counter() - t0
    print(f"frame {f} {1e3 * dt:8.1f} ms admm {st['admm_iterations']:3d} newton {st['newton_iterations']:5d} "
          f"ls {st['line_search_steps']:4d} pcg {st['pcg_iterations']:6d} contacts {st['max_contacts']} "
          f"attempts {st['attempts']}", flush=True)
