"""300-frame consensus runs at several PCG tolerances: where the line search
collapses (diagnostic for DESIGN 6b)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_15875_b200 import api  # noqa: E402
from paper_2605_15875_b200.scene import make_scenario  # noqa: E402

for spec in sys.argv[1:]:
    name, w = spec.split(":")
    for tol, mx in ((1e-10, 4000), (1e-12, 20000)):
        ctx = api.Context(api.Scene(make_scenario(name)), num_workers=int(w), pcg_rel_tol=tol, pcg_max_iters=mx)
        res = "ok"
        for f in range(300):
            try:
                ctx.run_frames(1)
            except Exception as e:  # noqa: BLE001
                res = f"frame {f}: {str(e)[:60]}"
                break
        print(json.dumps({"scene": name, "tol": tol, "result": res}), flush=True)
