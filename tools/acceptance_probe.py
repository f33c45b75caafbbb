"""Acceptance criteria 2, 3, 5 (proj/tests/acceptance.cpp) on the device at
two PCG tolerances, with per-scene detail (diagnostic tool)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2605_15875_b200 import api  # noqa: E402
from paper_2605_15875_b200.scene import make_scenario  # noqa: E402


def main():
    for tol in (1e-10, 1e-12):
        solver = dict(pcg_rel_tol=tol, pcg_max_iters=20000)
        sd = make_scenario("funnel-analog")
        ref = api.run_reference(sd, 100, **solver)
        run = api.run_distributed(sd, 2, 100, **solver)
        dyn = ~api.Scene(sd).is_static
        mse = [float(np.mean((run.q[f][dyn] - ref.q[f][dyn]) ** 2)) for f in range(100)]
        print(json.dumps({"tol": tol, "crit2_max_mse": max(mse), "argmax": int(np.argmax(mse)),
                          "mean_admm": float(np.mean([s["admm_iterations"] for s in run.stats]))}), flush=True)
        for d in [10, 100, 1000, 10000, 100000]:
            sd = make_scenario(f"density-sweep-{d}")
            a = np.mean([s["admm_iterations"] for s in api.run_distributed(sd, 2, 60, **solver).stats])
            sd.adapt.adapt_enabled = False
            f = np.mean([s["admm_iterations"] for s in api.run_distributed(sd, 2, 60, **solver).stats])
            print(json.dumps({"tol": tol, "density": d, "adaptive": a, "fixed": f, "reduction": 1 - a / f}), flush=True)
    for name in ["funnel-analog", "drop-grid-1", "drop-grid-2", "drop-grid-4", "density-sweep-10",
                 "density-sweep-100", "density-sweep-1000", "density-sweep-10000",
                 "density-sweep-100000", "blocked-merge", "heterogeneous"]:
        sd = make_scenario(name)
        workers = {"drop-grid-1": 1, "drop-grid-4": 4}.get(name, 2)
        ctx = api.Context(api.Scene(sd), num_workers=workers)
        msg = "ok"
        for f in range(300):
            try:
                ctx.run_frames(1)
            except Exception as e:  # noqa: BLE001
                msg = f"frame {f}: {e}"
                break
        print(json.dumps({"scene": name, "workers": workers, "result": msg}), flush=True)


if __name__ == "__main__":
    main()
