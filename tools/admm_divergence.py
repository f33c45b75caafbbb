"""Frame-by-frame GPU vs oracle comparison of a consensus-ADMM run: ADMM
count, attempts, h and max |q_gpu - q_oracle| per frame (diagnostic)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from paper_2605_15875_b200 import api  # noqa: E402
from paper_2605_15875_b200.scene import make_scenario  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "funnel-analog"
    workers = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    frames = int(sys.argv[3]) if len(sys.argv) > 3 else 100
    sd = make_scenario(name)
    ref = O.Scene(sd).run(frames, workers=workers)
    gpu = api.run_distributed(sd, workers, frames, pcg_rel_tol=1e-12, pcg_max_iters=20000)
    for f in range(frames):
        d = float(np.abs(gpu.q[f] - ref["q"][f]).max())
        print(json.dumps({"f": f, "admm_gpu": gpu.stats[f]["admm_iterations"], "admm_ref": int(ref["admm"][f]),
                          "att_gpu": gpu.stats[f]["attempts"], "att_ref": int(ref["attempts"][f]),
                          "h_gpu": gpu.h[f], "h_ref": float(ref["h"][f]), "maxdq": d}))
    # trace rows of the first differing frame
    tg, to = gpu.trace, ref["trace"]
    n = min(len(tg), len(to))
    for i in range(n):
        if tg[i][2] != to[i][2] or tg[i][0] != to[i][0] or abs(tg[i][3] - to[i][3]) > 1e-6 * max(abs(to[i][3]), 1e-30):
            print("first trace difference at row", i)
            for j in range(max(0, i - 2), min(n, i + 3)):
                print("gpu", list(np.round(tg[j], 12)))
                print("ref", list(np.round(to[j], 12)))
            break


if __name__ == "__main__":
    main()
