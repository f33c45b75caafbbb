"""Effect of the PCG relative tolerance on Newton/PCG work and on the state
(pile-1k, run_reference semantics), against a 1e-12 reference run."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_15875_b200 import api
from paper_2605_15875_b200.scene import make_scenario

scene = sys.argv[1] if len(sys.argv) > 1 else "pile-1k"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 30
sd = make_scenario(scene)
runs = {}
for tol in (1e-12, 1e-10, 1e-8, 1e-6, 1e-5, 1e-4, 1e-3):
    ctx = api.Context(api.Scene(sd), device=0, num_workers=0, pcg_rel_tol=tol, pcg_max_iters=20000)
    t0 = time.perf_counter()
    st = ctx.run_frames(frames)
    dt = time.perf_counter() - t0
    q, _ = ctx.state()
    runs[tol] = q
    ref = runs[1e-12]
    err = np.abs(q - ref).max()
    print(f"tol {tol:7.0e}: {1e3 * dt / frames:7.2f} ms/frame newton {sum(s['newton_iterations'] for s in st):6d} "
          f"pcg {sum(s['pcg_iterations'] for s in st):8d} admm {sum(s['admm_iterations'] for s in st):4d} "
          f"max|q-q_ref| {err:.3e}", flush=True)
