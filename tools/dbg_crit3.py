"""A 300-frame consensus-ADMM run per solver setting: where (if) the Newton
line search collapses, and the PCG iteration maxima before it (diagnostic)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_15875_b200 import api  # noqa: E402
from paper_2605_15875_b200.scene import make_scenario  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "drop-grid-2"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 100
for tol, mx in ((1e-10, 4000), (1e-12, 20000), (1e-14, 100000)):
    ctx = api.Context(api.Scene(make_scenario(name)), num_workers=2, pcg_rel_tol=tol, pcg_max_iters=mx)
    res, pmax = "ok", 0
    for f in range(frames):
        try:
            st = ctx.run_frames(1)[0]
            pmax = max(pmax, st["pcg_iterations"] / max(st["newton_iterations"], 1))
        except Exception as e:  # noqa: BLE001
            res = f"frame {f}: {e}"
            break
    print(json.dumps({"scene": name, "tol": tol, "max_iters": mx, "result": res, "max_mean_pcg_per_newton": pmax}), flush=True)
